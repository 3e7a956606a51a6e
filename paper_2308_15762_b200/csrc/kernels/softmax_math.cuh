// Softmax arithmetic shared by the fused attention kernels (sm_100a):
// SFU 2^x, packed f32x2 FMA / add / mul (FFMA2, FADD2, FMUL2: half the issue
// slots of the scalar forms), the 3-input max (FMNMX3) and a 2^x on the FMA
// pipe for the share of a tile the SFU cannot keep up with.
#pragma once

#include <cuda_runtime.h>

namespace wpk {
namespace smx {

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed f32x2 arithmetic (FFMA2 / FADD2): half the issue slots of the
// scalar forms for the softmax's per-element scale, sums and polynomial.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 a, b, c, d;\n"
      "mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5}; mov.b64 c, {%6, %7};\n"
      "fma.rn.f32x2 d, a, b, c;\n"
      "mov.b64 {%0, %1}, d;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 a, b, d;\n"
      "mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5};\n"
      "mul.rn.f32x2 d, a, b;\n"
      "mov.b64 {%0, %1}, d;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 a, b, d;\n"
      "mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5};\n"
      "add.rn.f32x2 d, a, b;\n"
      "mov.b64 {%0, %1}, d;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x for a pair on the FMA pipe instead of the SFU (which a 128 x 128 tile
// saturates as much as the tensor core): x = j + f with j = round(x) (the
// 1.5 * 2^23 shifter), 2^f by a degree-3 relative-minimax polynomial on
// [-1/2, 1/2] (max rel. error 7.5e-5, far below the bf16 rounding of P),
// 2^j added to the exponent field.  x <= 8 (lazy rescale); clamped at -126 so
// the exponent field never borrows into the sign (2^-126 ~ 0 after bf16).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  constexpr float kShift = 12582912.0f;  // 1.5 * 2^23
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = fadd2(x, make_float2(kShift, kShift));
  const float2 f = fadd2(x, fadd2(make_float2(kShift, kShift), make_float2(-t.x, -t.y)));
  float2 p = ffma2(make_float2(0.05517132f, 0.05517132f), f, make_float2(0.24261054f, 0.24261054f));
  p = ffma2(p, f, make_float2(0.69326097f, 0.69326097f));
  p = ffma2(p, f, make_float2(0.9999281f, 0.9999281f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

}  // namespace smx
}  // namespace wpk
