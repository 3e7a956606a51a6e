// HBM-bound kernels of the transformer stage: embedding, LayerNorm, attention
// softmax, fused cross-entropy, bias-gradient reduction, optimizer, init.
// Vectorised 16-byte accesses where the row is contiguous, one warp per row
// for row-wise reductions (warp shuffles, no shared memory), block-level
// partial sums + one global atomic per column for parameter gradients.
#include <cstdlib>
#include <type_traits>
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

#include "kernels/gemm.cuh"
#include "kernels/ops.cuh"
#include "kernels/softmax_math.cuh"

namespace wpk {
namespace {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(bf16 x) { return __bfloat162float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// 8 contiguous elements <-> 8 floats (16 B for bf16, 32 B for fp32).
__device__ __forceinline__ void load8(const float* p, float* v) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load8(const bf16* p, float* v) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const bf16* h = reinterpret_cast<const bf16*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __bfloat162float(h[i]);
}
__device__ __forceinline__ void store8(float* p, const float* v) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void store8(bf16* p, const float* v) {
  uint4 u;
  bf16* h = reinterpret_cast<bf16*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = __float2bfloat16_rn(v[i]);
  *reinterpret_cast<uint4*>(p) = u;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ embedding
template <typename T>
__global__ void embed_fwd_k(const int32_t* tok, const T* wte, const T* wpe, T* x, int T_, int seq, int h) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (i >= static_cast<int64_t>(T_) * h) return;
  const int t = static_cast<int>(i / h), c = static_cast<int>(i % h);
  float a[8], b[8];
  load8(wte + static_cast<int64_t>(tok[t]) * h + c, a);
  load8(wpe + static_cast<int64_t>(t % seq) * h + c, b);
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] += b[k];
  store8(x + i, a);
}

template <typename T>
__global__ void embed_bwd_k(const int32_t* tok, const T* dx, float* dwte, float* dwpe, int T_, int seq, int h) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (i >= static_cast<int64_t>(T_) * h) return;
  const int t = static_cast<int>(i / h), c = static_cast<int>(i % h);
  float g[8];
  load8(dx + i, g);
  float* pw = dwte + static_cast<int64_t>(tok[t]) * h + c;
  float* pp = dwpe + static_cast<int64_t>(t % seq) * h + c;
  // 16-byte vector atomics (sm_90+): 4 red operations instead of 16
  atomicAdd(reinterpret_cast<float4*>(pw), make_float4(g[0], g[1], g[2], g[3]));
  atomicAdd(reinterpret_cast<float4*>(pw + 4), make_float4(g[4], g[5], g[6], g[7]));
  atomicAdd(reinterpret_cast<float4*>(pp), make_float4(g[0], g[1], g[2], g[3]));
  atomicAdd(reinterpret_cast<float4*>(pp + 4), make_float4(g[4], g[5], g[6], g[7]));
}

// ------------------------------------------------------------------ layernorm
// Lane l owns columns {l*8 + 256*c + j}: C = h/256 chunks of 8.
template <typename T, int C>
__global__ void __launch_bounds__(256) ln_fwd_k(const T* x, const float* w, const float* b, T* y, float* mean,
                                                float* rstd, int T_, int h) {
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= T_) return;
  const T* xr = x + static_cast<int64_t>(row) * h;
  float v[C][8];
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    load8(xr + c * 256 + lane * 8, v[c]);
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[c][k];
  }
  const float mu = warp_sum(s) / h;
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c)
#pragma unroll
    for (int k = 0; k < 8; ++k) q += (v[c][k] - mu) * (v[c][k] - mu);
  const float rs = rsqrtf(warp_sum(q) / h + 1e-5f);
  T* yr = y + static_cast<int64_t>(row) * h;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int col = c * 256 + lane * 8;
    float wv[8], bv[8], o[8];
    load8(w + col, wv);
    load8(b + col, bv);
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = (v[c][k] - mu) * rs * wv[k] + bv[k];
    store8(yr + col, o);
  }
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

// bf16 forward, persistent warps over rows with the next row's loads in
// flight while the current one is reduced and written (the row kernel above
// is load-latency bound).  Same per-lane summation order as ln_fwd_k.
__device__ __forceinline__ void unpack8(const uint4& u, float* v) {
  const bf16* hv = reinterpret_cast<const bf16*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __bfloat162float(hv[i]);
}
template <int C>
__global__ void __launch_bounds__(256) ln_fwd_pipe_k(const bf16* x, const float* w, const float* b, bf16* y,
                                                     float* mean, float* rstd, int T_, int h) {
  const int lane = threadIdx.x % 32;
  const int nw = gridDim.x * (blockDim.x / 32);
  int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (row >= T_) return;
  uint4 cur[C], nxt[C];
#pragma unroll
  for (int c = 0; c < C; ++c)
    cur[c] = *reinterpret_cast<const uint4*>(x + static_cast<int64_t>(row) * h + c * 256 + lane * 8);
  for (; row < T_; row += nw) {
    if (row + nw < T_) {
#pragma unroll
      for (int c = 0; c < C; ++c)
        nxt[c] = *reinterpret_cast<const uint4*>(x + static_cast<int64_t>(row + nw) * h + c * 256 + lane * 8);
    }
    // Packed f32x2 arithmetic throughout (FADD2 / FFMA2 / FMUL2): the kernel
    // is issue-heavy next to its HBM traffic.
    float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&cur[c]);
#pragma unroll
      for (int k = 0; k < 4; ++k) s2 = smx::fadd2(s2, __bfloat1622float2(hv[k]));
    }
    const float mu = warp_sum(s2.x + s2.y) / h;
    const float2 nmu2 = make_float2(-mu, -mu);
    float2 q2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&cur[c]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 d = smx::fadd2(__bfloat1622float2(hv[k]), nmu2);
        q2 = smx::ffma2(d, d, q2);
      }
    }
    const float rs = rsqrtf(warp_sum(q2.x + q2.y) / h + 1e-5f);
    const float2 rs2 = make_float2(rs, rs);
    bf16* yr = y + static_cast<int64_t>(row) * h;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int col = c * 256 + lane * 8;
      const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&cur[c]);
      const float4 w0 = reinterpret_cast<const float4*>(w + col)[0], w1 = reinterpret_cast<const float4*>(w + col)[1];
      const float4 b0 = reinterpret_cast<const float4*>(b + col)[0], b1 = reinterpret_cast<const float4*>(b + col)[1];
      const float2 wv[4] = {make_float2(w0.x, w0.y), make_float2(w0.z, w0.w), make_float2(w1.x, w1.y),
                            make_float2(w1.z, w1.w)};
      const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                            make_float2(b1.z, b1.w)};
      uint4 u;
      __nv_bfloat162* ho = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 xh = smx::fmul2(smx::fadd2(__bfloat1622float2(hv[k]), nmu2), rs2);
        const float2 o = smx::ffma2(xh, wv[k], bv[k]);
        ho[k] = __floats2bfloat162_rn(o.x, o.y);
      }
      *reinterpret_cast<uint4*>(yr + col) = u;
    }
    if (lane == 0) {
      mean[row] = mu;
      rstd[row] = rs;
    }
#pragma unroll
    for (int c = 0; c < C; ++c) cur[c] = nxt[c];
  }
}

// dx: warp per row, two passes over the (L1-resident) row so no per-column
// state is held in registers.
template <typename T, int C>
__global__ void __launch_bounds__(256) ln_bwd_dx_k(const T* dy, const T* x, const float* mean, const float* rstd,
                                                   const float* w, const T* dres, T* dx, int T_, int h) {
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= T_) return;
  const int64_t off = static_cast<int64_t>(row) * h;
  const float mu = mean[row], rs = rstd[row];
  float sg = 0.f, sgx = 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int col = c * 256 + lane * 8;
    float d[8], xv[8], wv[8];
    load8(dy + off + col, d);
    load8(x + off + col, xv);
    load8(w + col, wv);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float g = d[k] * wv[k];
      sg += g;
      sgx += g * (xv[k] - mu) * rs;
    }
  }
  sg = warp_sum(sg) / h;
  sgx = warp_sum(sgx) / h;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int col = c * 256 + lane * 8;
    float d[8], xv[8], wv[8], r[8], o[8];
    load8(dy + off + col, d);
    load8(x + off + col, xv);
    load8(w + col, wv);
    if (dres) load8(dres + off + col, r);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      o[k] = rs * (d[k] * wv[k] - sg - (xv[k] - mu) * rs * sgx) + (dres ? r[k] : 0.f);
    store8(dx + off + col, o);
  }
}

// Fused LayerNorm backward: dx (as ln_bwd_dx_k) and the dw / db partial sums
// in one pass over dy and x.  A block owns a contiguous row range; each lane
// keeps its 8*C columns' dw / db sums in registers across the rows its warp
// visits, the 8 warps combine them through shared-memory atomics and the
// block adds its partial to the global fp32 gradients (one atomic per column
// per block).  HBM traffic per row: dy and x read once (the second pass hits
// L1), dx (and dres) once -- the separate dw/db kernel's re-read is gone.
template <typename T, int C>
__global__ void __launch_bounds__(256, 1) ln_bwd_fused_k(const T* dy, const T* x, const float* mean,
                                                         const float* rstd, const float* w, const T* dres, T* dx,
                                                         float* dw, float* db, int T_, int h, int rows_per) {
  extern __shared__ float red[];  // [2][h]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 2 * h; i += blockDim.x) red[i] = 0.f;
  float aw[C][8], ab[C][8];
#pragma unroll
  for (int c = 0; c < C; ++c)
#pragma unroll
    for (int k = 0; k < 8; ++k) aw[c][k] = ab[c][k] = 0.f;
  const int r0 = blockIdx.x * rows_per, r1 = min(T_, r0 + rows_per);
  for (int row = r0 + warp; row < r1; row += 8) {
    const int64_t off = static_cast<int64_t>(row) * h;
    const float mu = mean[row], rs = rstd[row];
    float sg = 0.f, sgx = 0.f;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int col = c * 256 + lane * 8;
      float d[8], xv[8], wv[8];
      load8(dy + off + col, d);
      load8(x + off + col, xv);
      load8(w + col, wv);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float g = d[k] * wv[k];
        sg += g;
        sgx += g * (xv[k] - mu) * rs;
      }
    }
    sg = warp_sum(sg) / h;
    sgx = warp_sum(sgx) / h;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int col = c * 256 + lane * 8;
      float d[8], xv[8], wv[8], r[8], o[8];
      load8(dy + off + col, d);
      load8(x + off + col, xv);
      load8(w + col, wv);
      if (dres) load8(dres + off + col, r);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float xh = (xv[k] - mu) * rs;
        o[k] = rs * (d[k] * wv[k] - sg - xh * sgx) + (dres ? r[k] : 0.f);
        aw[c][k] += d[k] * xh;
        ab[c][k] += d[k];
      }
      store8(dx + off + col, o);
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < C; ++c)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      atomicAdd(&red[c * 256 + lane * 8 + k], aw[c][k]);
      atomicAdd(&red[h + c * 256 + lane * 8 + k], ab[c][k]);
    }
  __syncthreads();
  if (r0 < r1)
    for (int i = threadIdx.x; i < h; i += blockDim.x) {
      atomicAdd(&dw[i], red[i]);
      atomicAdd(&db[i], red[h + i]);
    }
}

// Column-owned LayerNorm backward: a block of h/8 threads spans one row (each
// thread owns 8 contiguous columns -> one 16-byte access per tensor per row)
// and walks a contiguous row range R = 4 rows at a time.  The row sums
// (sum g, sum g*xhat with g = dy*w) are block reductions -- warp shuffles,
// then one smem exchange per 4 rows -- and each thread keeps only its 8
// columns' dw / db sums, so registers stay low, several blocks share an SM
// and dy / x stream from HBM exactly once (kept in registers between the
// reduction and the dx update).
constexpr int LNR = 4;
template <typename T>
__global__ void __launch_bounds__(512, 1) ln_bwd_cols_k(const T* dy, const T* x, const float* mean, const float* rstd,
                                                      const float* w, const T* dres, T* dx, float* dw, float* db,
                                                      int T_, int h, int rows_per) {
  __shared__ float red[32][2 * LNR];
  __shared__ float tot[2 * LNR];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  const int col = threadIdx.x * 8;
  float wv[8], aw[8], ab[8];
  load8(w + col, wv);
#pragma unroll
  for (int k = 0; k < 8; ++k) aw[k] = ab[k] = 0.f;
  const int r0 = blockIdx.x * rows_per, r1 = min(T_, r0 + rows_per);
  const float inv_h = 1.f / h;
  for (int rb = r0; rb < r1; rb += LNR) {
    float d[LNR][8], xh[LNR][8], part[2 * LNR];
#pragma unroll
    for (int i = 0; i < LNR; ++i) {
      const int row = rb + i;
      part[2 * i] = part[2 * i + 1] = 0.f;
      if (row < r1) {
        const int64_t off = static_cast<int64_t>(row) * h + col;
        load8(dy + off, d[i]);
        load8(x + off, xh[i]);
        const float mu = mean[row], rs = rstd[row];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          xh[i][k] = (xh[i][k] - mu) * rs;
          const float g = d[i][k] * wv[k];
          part[2 * i] += g;
          part[2 * i + 1] += g * xh[i][k];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 2 * LNR; ++q) part[q] = warp_sum(part[q]);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 2 * LNR; ++q) red[warp][q] = part[q];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int q = 0; q < 2 * LNR; ++q) {
        float v = lane < nw ? red[lane][q] : 0.f;
        v = warp_sum(v);
        if (lane == 0) tot[q] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < LNR; ++i) {
      const int row = rb + i;
      if (row >= r1) break;
      const int64_t off = static_cast<int64_t>(row) * h + col;
      const float rs = rstd[row], sg = tot[2 * i] * inv_h, sgx = tot[2 * i + 1] * inv_h;
      float r[8], o[8];
      if (dres) load8(dres + off, r);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        o[k] = rs * (d[i][k] * wv[k] - sg - xh[i][k] * sgx) + (dres ? r[k] : 0.f);
        aw[k] += d[i][k] * xh[i][k];
        ab[k] += d[i][k];
      }
      store8(dx + off, o);
    }
  }
  if (r0 < r1)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      atomicAdd(&dw[col + k], aw[k]);
      atomicAdd(&db[col + k], ab[k]);
    }
}

// Elementwise LayerNorm dx from precomputed row sums (see ops.cuh): 8
// contiguous elements per thread, 16-byte accesses, grid-stride.
template <typename T>
__global__ void __launch_bounds__(256) ln_bwd_dx_rows_k(const T* dy, const T* x, const float* mean,
                                                        const float* rstd, const float* w, const float* rows,
                                                        const T* dres, T* dx, int64_t n8, int h) {
  const float inv_h = 1.f / h;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t off = i * 8;
    const int row = static_cast<int>(off / h), col = static_cast<int>(off % h);
    float d[8], xv[8], wv[8], r[8], o[8];
    load8(dy + off, d);
    load8(x + off, xv);
    load8(w + col, wv);
    if (dres) load8(dres + off, r);
    const float mu = mean[row], rs = rstd[row], sg = rows[2 * row] * inv_h, sgx = rows[2 * row + 1] * inv_h;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float xh = (xv[k] - mu) * rs;
      o[k] = rs * (d[k] * wv[k] - sg - xh * sgx) + (dres ? r[k] : 0.f);
    }
    store8(dx + off, o);
  }
}

// Same dx, blocked 64 columns x 128 rows per CTA so the column sums of dx
// (the bias gradient of the unit below: attention projection or FC2) come
// out of the same pass: 32 row-partials per column meet in shared memory,
// one atomic per column per block.
template <typename T>
__device__ __forceinline__ float round_to_t(float v) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(__float2bfloat16_rn(v));
  else return v;
}
template <typename T>
__global__ void __launch_bounds__(256) ln_bwd_dx_rows_cs_k(const T* dy, const T* x, const float* mean,
                                                           const float* rstd, const float* w, const float* rows,
                                                           const T* dres, T* dx, float* dcol, int T_, int h) {
  __shared__ float part[32][65];
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const int col = blockIdx.x * 64 + tx * 8;
  const int t0 = blockIdx.y * 128;
  const float inv_h = 1.f / h;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (col < h) {
    float wv[8];
    load8(w + col, wv);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int row = t0 + ty + 32 * k;
      if (row >= T_) break;
      const int64_t off = static_cast<int64_t>(row) * h + col;
      const float mu = mean[row], rs = rstd[row], sg = rows[2 * row] * inv_h, sgx = rows[2 * row + 1] * inv_h;
      if constexpr (std::is_same_v<T, bf16>) {
        // bf16: packed f32x2 arithmetic (half the FP32 issue slots)
        const uint4 ud = *reinterpret_cast<const uint4*>(dy + off), ux = *reinterpret_cast<const uint4*>(x + off);
        const uint4 ur = dres ? *reinterpret_cast<const uint4*>(dres + off) : make_uint4(0u, 0u, 0u, 0u);
        const __nv_bfloat162* hd = reinterpret_cast<const __nv_bfloat162*>(&ud);
        const __nv_bfloat162* hx = reinterpret_cast<const __nv_bfloat162*>(&ux);
        const __nv_bfloat162* hr = reinterpret_cast<const __nv_bfloat162*>(&ur);
        const float2 nmu2 = make_float2(-mu, -mu), rs2 = make_float2(rs, rs);
        const float2 nsg2 = make_float2(-sg, -sg), nsgx2 = make_float2(-sgx, -sgx);
        uint4 uo;
        __nv_bfloat162* ho = reinterpret_cast<__nv_bfloat162*>(&uo);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 xh = smx::fmul2(smx::fadd2(__bfloat1622float2(hx[k]), nmu2), rs2);
          float2 t = smx::ffma2(__bfloat1622float2(hd[k]), make_float2(wv[2 * k], wv[2 * k + 1]), nsg2);
          t = smx::ffma2(xh, nsgx2, t);
          const float2 o = smx::ffma2(t, rs2, __bfloat1622float2(hr[k]));
          ho[k] = __floats2bfloat162_rn(o.x, o.y);
          const float2 orr = __bfloat1622float2(ho[k]);
          acc[2 * k] += orr.x;
          acc[2 * k + 1] += orr.y;
        }
        *reinterpret_cast<uint4*>(dx + off) = uo;
      } else {
        float d[8], xv[8], r[8], o[8];
        load8(dy + off, d);
        load8(x + off, xv);
        if (dres) load8(dres + off, r);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (xv[j] - mu) * rs;
          o[j] = rs * (d[j] * wv[j] - sg - xh * sgx) + (dres ? r[j] : 0.f);
        }
        store8(dx + off, o);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += round_to_t<T>(o[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) part[ty][tx * 8 + j] = acc[j];
  __syncthreads();
  if (threadIdx.x < 64 && blockIdx.x * 64 + static_cast<int>(threadIdx.x) < h) {
    float sum = 0.f;
#pragma unroll 8
    for (int y = 0; y < 32; ++y) sum += part[y][threadIdx.x];
    atomicAdd(dcol + blockIdx.x * 64 + threadIdx.x, sum);
  }
}

// dw, db: lane <-> column (coalesced), 8 warps stride over a row range, block
// partials reduced in shared memory, one atomic per column per block.
template <typename T>
__global__ void __launch_bounds__(256) ln_bwd_dwdb_k(const T* dy, const T* x, const float* mean, const float* rstd,
                                                     float* dw, float* db, int T_, int h, int rows_per) {
  __shared__ float sw[8][33], sb[8][33];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int col = blockIdx.x * 32 + lane;
  const int r0 = blockIdx.y * rows_per, r1 = min(T_, r0 + rows_per);
  float aw = 0.f, ab = 0.f;
  if (col < h) {
    for (int r = r0 + warp; r < r1; r += 8) {
      const int64_t o = static_cast<int64_t>(r) * h + col;
      const float d = to_f(dy[o]);
      aw += d * (to_f(x[o]) - mean[r]) * rstd[r];
      ab += d;
    }
  }
  sw[warp][lane] = aw;
  sb[warp][lane] = ab;
  __syncthreads();
  if (warp == 0 && col < h) {
    float tw = 0.f, tb = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      tw += sw[i][lane];
      tb += sb[i][lane];
    }
    atomicAdd(&dw[col], tw);
    atomicAdd(&db[col], tb);
  }
}

// ------------------------------------------------------------------- softmax
// Warp per row; lane l holds columns l + 32*k.
// Causal rows only touch columns j <= q; P is written up to the end of q's
// 128-wide tile (zeros past the diagonal) -- exactly the K range the causal
// P.V / dS.K GEMMs read (kCausalKUpToRow) -- and not beyond.
template <typename T>
__global__ void __launch_bounds__(256) softmax_fwd_k(const float* S, T* P, int rows, int n, int causal) {
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= rows) return;
  const int q = row % n;
  const int valid = causal ? q + 1 : n;
  const int lim = causal ? min(n, (q / 128 + 1) * 128) : n;
  const float* sr = S + static_cast<int64_t>(row) * n;
  T* pr = P + static_cast<int64_t>(row) * n;
  float v[32];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const int j = lane + 32 * k;
    v[k] = j < valid ? sr[j] : -INFINITY;
    m = fmaxf(m, v[k]);
  }
  m = warp_max(m);
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    v[k] = (v[k] == -INFINITY) ? 0.f : __expf(v[k] - m);
    s += v[k];
  }
  const float inv = 1.f / warp_sum(s);
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const int j = lane + 32 * k;
    if (j < lim) pr[j] = from_f<T>(v[k] * inv);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) softmax_bwd_k(const float* dP, T* P, int rows, int n, float scale,
                                                     int causal) {
  const int row = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (row >= rows) return;
  const int q = row % n;
  const int valid = causal ? q + 1 : n;
  const int lim = causal ? min(n, (q / 128 + 1) * 128) : n;
  const float* dr = dP + static_cast<int64_t>(row) * n;
  T* pr = P + static_cast<int64_t>(row) * n;
  float p[32], d[32];
  float dot = 0.f;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const int j = lane + 32 * k;
    p[k] = j < valid ? to_f(pr[j]) : 0.f;
    d[k] = j < valid ? dr[j] : 0.f;
    dot += p[k] * d[k];
  }
  dot = warp_sum(dot);
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const int j = lane + 32 * k;
    if (j < lim) pr[j] = from_f<T>(scale * p[k] * (d[k] - dot));
  }
}

// -------------------------------------------------------------- cross-entropy
template <typename T>
__global__ void __launch_bounds__(256) xent_k(T* logits, const int32_t* labels, float* loss, int V, float loss_scale,
                                              float grad_scale) {
  const int row = blockIdx.x;
  T* lr = logits + static_cast<int64_t>(row) * V;
  float m = -INFINITY, s = 0.f;
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    const float x = to_f(lr[j]);
    if (x > m) {
      s = s * __expf(m - x) + 1.f;
      m = x;
    } else {
      s += __expf(x - m);
    }
  }
  __shared__ float sm[32], ss[32];
  // warp combine of (m, s)
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float mm = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
    m = mm;
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
    sm[warp] = m;
    ss[warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x / 32;
    m = lane < nw ? sm[lane] : -INFINITY;
    s = lane < nw ? ss[lane] : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
      const float mm = fmaxf(m, m2);
      s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
      m = mm;
    }
    if (lane == 0) {
      sm[0] = m + logf(s);  // lse
    }
  }
  __syncthreads();
  const float lse = sm[0];
  const int label = labels[row];
  if (threadIdx.x == 0) atomicAdd(loss, (lse - to_f(lr[label])) * loss_scale);
  __syncthreads();  // the label logit is read before being overwritten
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    const float p = __expf(to_f(lr[j]) - lse);
    lr[j] = from_f<T>((p - (j == label ? 1.f : 0.f)) * grad_scale);
  }
}

// Vectorised cross-entropy: XR rows per 256-thread block, 16-byte accesses.
// Pass 1 keeps a running (max, sum) per thread, rescaling once per 8-vector
// instead of per element; pass 2 rewrites the row with (softmax - onehot) *
// grad_scale (the row, 100 KB at V = 50304, is still in L2).  One loss atomic
// per block.  Needs V % 8 == 0.
constexpr int XR = 4;
template <typename T>
__global__ void __launch_bounds__(256) xent_vec_k(T* logits, const int32_t* labels, float* loss, int T_, int V,
                                                  float loss_scale, float grad_scale) {
  __shared__ float sm[32], ss[32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  constexpr float L2E = 1.4426950408889634f;
  float block_loss = 0.f;
  for (int rr = 0; rr < XR; ++rr) {
    const int row = blockIdx.x * XR + rr;
    if (row >= T_) break;
    T* lr = logits + static_cast<int64_t>(row) * V;
    float m = -INFINITY, sum = 0.f;
    for (int j = threadIdx.x * 8; j < V; j += blockDim.x * 8) {
      float v[8];
      load8(lr + j, v);
      float mx = v[0];
#pragma unroll
      for (int k = 1; k < 8; ++k) mx = fmaxf(mx, v[k]);
      if (mx > m) {
        sum *= exp2f((m - mx) * L2E);
        m = mx;
      }
      const float mb = m * L2E;
#pragma unroll
      for (int k = 0; k < 8; ++k) sum += exp2f(fmaf(v[k], L2E, -mb));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
      const float mm = fmaxf(m, m2);
      sum = (m == -INFINITY ? 0.f : sum * exp2f((m - mm) * L2E)) + (m2 == -INFINITY ? 0.f : s2 * exp2f((m2 - mm) * L2E));
      m = mm;
    }
    if (lane == 0) {
      sm[warp] = m;
      ss[warp] = sum;
    }
    __syncthreads();
    if (warp == 0) {
      m = lane < nw ? sm[lane] : -INFINITY;
      sum = lane < nw ? ss[lane] : 0.f;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
        const float mm = fmaxf(m, m2);
        sum = (m == -INFINITY ? 0.f : sum * exp2f((m - mm) * L2E)) +
              (m2 == -INFINITY ? 0.f : s2 * exp2f((m2 - mm) * L2E));
        m = mm;
      }
      if (lane == 0) sm[0] = m + logf(sum);  // lse
    }
    __syncthreads();
    const float lse = sm[0];
    const int label = labels[row];
    if (threadIdx.x == 0) block_loss += lse - to_f(lr[label]);
    __syncthreads();  // the label logit is read before being overwritten; sm reused next row
    const float lb = lse * L2E;
    for (int j = threadIdx.x * 8; j < V; j += blockDim.x * 8) {
      float v[8];
      load8(lr + j, v);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = (exp2f(fmaf(v[k], L2E, -lb)) - (j + k == label ? 1.f : 0.f)) * grad_scale;
      store8(lr + j, v);
    }
  }
  if (threadIdx.x == 0) atomicAdd(loss, block_loss * loss_scale);
}

// --------------------------------------------------------------- bias grads
// Block = 8 warps over a 256-column strip; lane owns 8 contiguous columns
// (one 16-byte load per row for bf16), warps stride over the block's rows,
// partials reduced through shared memory, one atomic per column per block.
template <typename T>
__global__ void __launch_bounds__(256) colsum_k(const T* dy, float* db, int T_, int n, int ld, int rows_per) {
  __shared__ float red[8][256];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int col = blockIdx.x * 256 + lane * 8;
  const int r0 = blockIdx.y * rows_per, r1 = min(T_, r0 + rows_per);
  float acc[8] = {};
  if (col < n) {
    for (int r = r0 + warp; r < r1; r += 8) {
      float v[8];
      load8(dy + static_cast<int64_t>(r) * ld + col, v);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += v[k];
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) red[warp][lane * 8 + k] = acc[k];
  __syncthreads();
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c < n) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][threadIdx.x];
    atomicAdd(&db[c], t);
  }
}

// ---------------------------------------------------------------- optimizer
__device__ __forceinline__ float optim_one(const OptimArgs& a, float p, float gr, float& mi, float& vi, float bc1,
                                           float bc2) {
  if (a.kind == 0) return p - a.lr * (gr + a.weight_decay * p);
  mi = a.beta1 * mi + (1.f - a.beta1) * gr;
  vi = a.beta2 * vi + (1.f - a.beta2) * gr * gr;
  return p - a.lr * ((mi / bc1) / (sqrtf(vi / bc2) + a.eps) + a.weight_decay * p);
}

// Fused SGD / AdamW + bf16 shadow refresh + gradient zeroing: 16-byte
// accesses over four parameters per thread (34 B per parameter moved).
__global__ void optim_k(OptimArgs a, float* w, float* g, float* m, float* v, bf16* shadow, int64_t n, float bc1,
                        float bc2) {
  const int64_t n4 = n / 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 p = reinterpret_cast<float4*>(w)[i];
    const float4 gr = reinterpret_cast<const float4*>(g)[i];
    float4 mi = make_float4(0.f, 0.f, 0.f, 0.f), vi = mi;
    if (a.kind != 0) {
      mi = reinterpret_cast<float4*>(m)[i];
      vi = reinterpret_cast<float4*>(v)[i];
    }
    p.x = optim_one(a, p.x, gr.x, mi.x, vi.x, bc1, bc2);
    p.y = optim_one(a, p.y, gr.y, mi.y, vi.y, bc1, bc2);
    p.z = optim_one(a, p.z, gr.z, mi.z, vi.z, bc1, bc2);
    p.w = optim_one(a, p.w, gr.w, mi.w, vi.w, bc1, bc2);
    if (a.kind != 0) {
      reinterpret_cast<float4*>(m)[i] = mi;
      reinterpret_cast<float4*>(v)[i] = vi;
    }
    reinterpret_cast<float4*>(w)[i] = p;
    reinterpret_cast<float4*>(g)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (shadow) {
      uint2 u;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
      h[0] = __floats2bfloat162_rn(p.x, p.y);
      h[1] = __floats2bfloat162_rn(p.z, p.w);
      reinterpret_cast<uint2*>(shadow)[i] = u;
    }
  }
  for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    float mi = a.kind != 0 ? m[i] : 0.f, vi = a.kind != 0 ? v[i] : 0.f;
    const float p = optim_one(a, w[i], g[i], mi, vi, bc1, bc2);
    if (a.kind != 0) m[i] = mi, v[i] = vi;
    w[i] = p;
    g[i] = 0.f;
    if (shadow) shadow[i] = __float2bfloat16_rn(p);
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void init_normal_k(float* p, int64_t n, float std, uint64_t seed) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = mix64(seed ^ mix64(static_cast<uint64_t>(i)));
    const float u1 = (static_cast<float>(r >> 40) + 1.f) * (1.f / 16777217.f);
    const float u2 = static_cast<float>((r >> 16) & 0xFFFFFF) * (1.f / 16777216.f);
    p[i] = std * sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
  }
}

__global__ void fill_k(float* p, int64_t n, float v) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

__global__ void cast_k(const float* s, bf16* d, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d[i] = __float2bfloat16_rn(s[i]);
}

int grid_for(int64_t n, int block, int cap = 148 * 16) {
  return static_cast<int>(std::min<int64_t>((n + block - 1) / block, cap));
}

int sm_count();

template <typename T>
int ln_fwd_dispatch(const T* x, const float* w, const float* b, T* y, float* mean, float* rstd, int T_, int h,
                    cudaStream_t s) {
  const dim3 grid((T_ + 7) / 8), block(256);
  static const bool pipe_off = std::getenv("WP_LN_FWD_ROWS") != nullptr;  // A/B switch
  if constexpr (std::is_same_v<T, bf16>) {
    if (!pipe_off && (h == 1024 || h == 2048)) {
      const int blocks = std::max(1, std::min((T_ + 7) / 8, 2 * sm_count()));  // 2 CTAs per SM fit (<= 128 regs)
      if (h == 1024) ln_fwd_pipe_k<4><<<blocks, block, 0, s>>>(x, w, b, y, mean, rstd, T_, h);
      else ln_fwd_pipe_k<8><<<blocks, block, 0, s>>>(x, w, b, y, mean, rstd, T_, h);
      check_launch("layernorm_fwd");
      return 1;
    }
  }
  // One instantiation per chunk count: every hidden size ModelSpec accepts
  // (a multiple of 256 up to 4096).
  switch (h / 256) {
#define WP_LN_FWD_CASE(c) \
  case c: ln_fwd_k<T, c><<<grid, block, 0, s>>>(x, w, b, y, mean, rstd, T_, h); break;
    WP_LN_FWD_CASE(1) WP_LN_FWD_CASE(2) WP_LN_FWD_CASE(3) WP_LN_FWD_CASE(4) WP_LN_FWD_CASE(5) WP_LN_FWD_CASE(6)
    WP_LN_FWD_CASE(7) WP_LN_FWD_CASE(8) WP_LN_FWD_CASE(9) WP_LN_FWD_CASE(10) WP_LN_FWD_CASE(11)
    WP_LN_FWD_CASE(12) WP_LN_FWD_CASE(13) WP_LN_FWD_CASE(14) WP_LN_FWD_CASE(15) WP_LN_FWD_CASE(16)
#undef WP_LN_FWD_CASE
    default: throw std::runtime_error("layernorm: hidden must be a multiple of 256, at most 4096");
  }
  check_launch("layernorm_fwd");
  return 1;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <typename T, int C>
void launch_ln_bwd_fused(const T* dy, const T* x, const float* mean, const float* rstd, const float* w,
                         const T* dres, T* dx, float* dw, float* db, int T_, int h, cudaStream_t s) {
  // One block per SM, each over a contiguous row range (a multiple of 8 rows).
  const int blocks = std::max(1, std::min(sm_count(), (T_ + 7) / 8));
  const int rows_per = ((T_ + blocks - 1) / blocks + 7) / 8 * 8;
  const int grid = (T_ + rows_per - 1) / rows_per;
  const size_t smem = 2 * size_t(h) * sizeof(float);
  ln_bwd_fused_k<T, C><<<grid, 256, smem, s>>>(dy, x, mean, rstd, w, dres, dx, dw, db, T_, h, rows_per);
}

template <typename T>
int ln_bwd_dispatch(const T* dy, const T* x, const float* mean, const float* rstd, const float* w, const T* dres,
                    T* dx, float* dw, float* db, int T_, int h, cudaStream_t s) {
  if (h % 256 == 0 && h / 8 <= 512) {
    // Two blocks per SM, contiguous row ranges (multiples of LNR rows).
    const int blocks = std::max(1, std::min(2 * sm_count(), (T_ + LNR - 1) / LNR));
    const int rows_per = ((T_ + blocks - 1) / blocks + LNR - 1) / LNR * LNR;
    const int grid = (T_ + rows_per - 1) / rows_per;
    ln_bwd_cols_k<T><<<grid, h / 8, 0, s>>>(dy, x, mean, rstd, w, dres, dx, dw, db, T_, h, rows_per);
    check_launch("layernorm_bwd (column-owned)");
    return 1;
  }
  bool fused = h % 256 == 0;
  switch (fused ? h / 256 : 0) {
    case 1: launch_ln_bwd_fused<T, 1>(dy, x, mean, rstd, w, dres, dx, dw, db, T_, h, s); break;
    case 2: launch_ln_bwd_fused<T, 2>(dy, x, mean, rstd, w, dres, dx, dw, db, T_, h, s); break;
    case 4: launch_ln_bwd_fused<T, 4>(dy, x, mean, rstd, w, dres, dx, dw, db, T_, h, s); break;
    case 8: launch_ln_bwd_fused<T, 8>(dy, x, mean, rstd, w, dres, dx, dw, db, T_, h, s); break;
    default: fused = false; break;  // h = 4096: dw/db sums would not fit in registers
  }
  if (fused) {
    check_launch("layernorm_bwd (fused)");
    return 1;
  }
  const dim3 grid((T_ + 7) / 8), block(256);
  switch (h / 256) {
    case 1: ln_bwd_dx_k<T, 1><<<grid, block, 0, s>>>(dy, x, mean, rstd, w, dres, dx, T_, h); break;
    case 2: ln_bwd_dx_k<T, 2><<<grid, block, 0, s>>>(dy, x, mean, rstd, w, dres, dx, T_, h); break;
    case 4: ln_bwd_dx_k<T, 4><<<grid, block, 0, s>>>(dy, x, mean, rstd, w, dres, dx, T_, h); break;
    case 8: ln_bwd_dx_k<T, 8><<<grid, block, 0, s>>>(dy, x, mean, rstd, w, dres, dx, T_, h); break;
    case 16: ln_bwd_dx_k<T, 16><<<grid, block, 0, s>>>(dy, x, mean, rstd, w, dres, dx, T_, h); break;
    default: throw std::runtime_error("layernorm: hidden must be 256 * {1,2,4,8,16}");
  }
  check_launch("layernorm_bwd_dx");
  const int rows_per = 256;
  const dim3 g2((h + 31) / 32, (T_ + rows_per - 1) / rows_per);
  ln_bwd_dwdb_k<T><<<g2, 256, 0, s>>>(dy, x, mean, rstd, dw, db, T_, h, rows_per);
  check_launch("layernorm_bwd_dwdb");
  return 2;
}

__global__ void wait_flag_k(const uint32_t* flag, uint32_t epoch, const volatile uint32_t* abort_word) {
  for (uint32_t it = 0;; ++it) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (static_cast<int32_t>(v - epoch) >= 0) return;
    if ((it & 15) == 15 && *abort_word) return;  // host memory: polled every 16th spin
    __nanosleep(256);
  }
}


// One-shot all-reduce (scaled sum) of this member's share; float4 granules,
// fixed summation order (member 0..G-1) so every member stores the same bits.
constexpr int kMaxGroup = 32;
__global__ void allreduce_scaled_k(float* const* bufs, int D, int64_t lo4, int64_t hi4, float scale) {
  float4* b[kMaxGroup];
  for (int r = 0; r < D; ++r) b[r] = reinterpret_cast<float4*>(bufs[r]);
  for (int64_t i = lo4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < hi4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 acc = b[0][i];
    for (int r = 1; r < D; ++r) {
      const float4 v = b[r][i];
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    }
    acc.x *= scale, acc.y *= scale, acc.z *= scale, acc.w *= scale;
    for (int r = 0; r < D; ++r) b[r][i] = acc;
  }
}

}  // namespace

#define WP_DISPATCH(dtype, F, ...) \
  ((dtype) == kBF16 ? F<bf16>(__VA_ARGS__) : F<float>(__VA_ARGS__))

int embed_fwd(int dtype, const int32_t* tok, const void* wte, const void* wpe, void* x, int T_, int seq, int h,
              cudaStream_t s) {
  if (h % 8) throw std::runtime_error("embed: hidden must be a multiple of 8");
  const int64_t n = static_cast<int64_t>(T_) * h / 8;
  const int grid = static_cast<int>((n + 255) / 256);
  if (dtype == kBF16)
    embed_fwd_k<bf16><<<grid, 256, 0, s>>>(tok, static_cast<const bf16*>(wte), static_cast<const bf16*>(wpe),
                                           static_cast<bf16*>(x), T_, seq, h);
  else
    embed_fwd_k<float><<<grid, 256, 0, s>>>(tok, static_cast<const float*>(wte), static_cast<const float*>(wpe),
                                            static_cast<float*>(x), T_, seq, h);
  check_launch("embed_fwd");
  return 1;
}

int embed_bwd(int dtype, const int32_t* tok, const void* dx, float* dwte, float* dwpe, int T_, int seq, int h,
              cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(T_) * h / 8;
  const int grid = static_cast<int>((n + 255) / 256);
  if (dtype == kBF16)
    embed_bwd_k<bf16><<<grid, 256, 0, s>>>(tok, static_cast<const bf16*>(dx), dwte, dwpe, T_, seq, h);
  else
    embed_bwd_k<float><<<grid, 256, 0, s>>>(tok, static_cast<const float*>(dx), dwte, dwpe, T_, seq, h);
  check_launch("embed_bwd");
  return 1;
}

int layernorm_fwd(int dtype, const void* x, const float* w, const float* b, void* y, float* mean, float* rstd, int T_,
                  int h, cudaStream_t s) {
  if (dtype == kBF16)
    return ln_fwd_dispatch<bf16>(static_cast<const bf16*>(x), w, b, static_cast<bf16*>(y), mean, rstd, T_, h, s);
  return ln_fwd_dispatch<float>(static_cast<const float*>(x), w, b, static_cast<float*>(y), mean, rstd, T_, h, s);
}

int layernorm_bwd(int dtype, const void* dy, const void* x, const float* mean, const float* rstd, const float* w,
                  const void* dres, void* dx, float* dw, float* db, int T_, int h, cudaStream_t s) {
  if (dtype == kBF16)
    return ln_bwd_dispatch<bf16>(static_cast<const bf16*>(dy), static_cast<const bf16*>(x), mean, rstd, w,
                                 static_cast<const bf16*>(dres), static_cast<bf16*>(dx), dw, db, T_, h, s);
  return ln_bwd_dispatch<float>(static_cast<const float*>(dy), static_cast<const float*>(x), mean, rstd, w,
                                static_cast<const float*>(dres), static_cast<float*>(dx), dw, db, T_, h, s);
}

int layernorm_bwd_dx_rows(int dtype, const void* dy, const void* x, const float* mean, const float* rstd,
                          const float* w, const float* rows, const void* dres, void* dx, int T_, int h,
                          cudaStream_t s, float* dcol) {
  if (h % 8) throw std::runtime_error("layernorm_bwd_dx_rows: hidden must be a multiple of 8");
  if (dcol) {
    const dim3 grid((h + 63) / 64, (T_ + 127) / 128);
    if (dtype == kBF16)
      ln_bwd_dx_rows_cs_k<bf16><<<grid, 256, 0, s>>>(static_cast<const bf16*>(dy), static_cast<const bf16*>(x), mean,
                                                     rstd, w, rows, static_cast<const bf16*>(dres),
                                                     static_cast<bf16*>(dx), dcol, T_, h);
    else
      ln_bwd_dx_rows_cs_k<float><<<grid, 256, 0, s>>>(static_cast<const float*>(dy), static_cast<const float*>(x),
                                                      mean, rstd, w, rows, static_cast<const float*>(dres),
                                                      static_cast<float*>(dx), dcol, T_, h);
    check_launch("layernorm_bwd_dx_rows");
    return 1;
  }
  const int64_t n8 = static_cast<int64_t>(T_) * h / 8;
  const int grid = static_cast<int>(std::min<int64_t>((n8 + 255) / 256, 8 * sm_count()));
  if (dtype == kBF16)
    ln_bwd_dx_rows_k<bf16><<<grid, 256, 0, s>>>(static_cast<const bf16*>(dy), static_cast<const bf16*>(x), mean,
                                                rstd, w, rows, static_cast<const bf16*>(dres), static_cast<bf16*>(dx),
                                                n8, h);
  else
    ln_bwd_dx_rows_k<float><<<grid, 256, 0, s>>>(static_cast<const float*>(dy), static_cast<const float*>(x), mean,
                                                 rstd, w, rows, static_cast<const float*>(dres),
                                                 static_cast<float*>(dx), n8, h);
  check_launch("layernorm_bwd_dx_rows");
  return 1;
}

int softmax_fwd(int dtype, const float* S, void* P, int rows, int n, int causal, cudaStream_t s) {
  if (n > 1024) throw std::runtime_error("softmax: row length must be <= 1024");
  const int grid = (rows + 7) / 8;
  if (dtype == kBF16) softmax_fwd_k<bf16><<<grid, 256, 0, s>>>(S, static_cast<bf16*>(P), rows, n, causal);
  else softmax_fwd_k<float><<<grid, 256, 0, s>>>(S, static_cast<float*>(P), rows, n, causal);
  check_launch("softmax_fwd");
  return 1;
}

int softmax_bwd(int dtype, const float* dP, void* P, int rows, int n, float scale, int causal, cudaStream_t s) {
  if (n > 1024) throw std::runtime_error("softmax: row length must be <= 1024");
  const int grid = (rows + 7) / 8;
  if (dtype == kBF16) softmax_bwd_k<bf16><<<grid, 256, 0, s>>>(dP, static_cast<bf16*>(P), rows, n, scale, causal);
  else softmax_bwd_k<float><<<grid, 256, 0, s>>>(dP, static_cast<float*>(P), rows, n, scale, causal);
  check_launch("softmax_bwd");
  return 1;
}

__global__ void stamp_globaltimer_k(uint64_t* out) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}

int stamp_globaltimer(uint64_t* out, cudaStream_t s) {
  stamp_globaltimer_k<<<1, 1, 0, s>>>(out);
  check_launch("stamp_globaltimer");
  return 1;
}

int wait_flag(cudaStream_t s, const uint32_t* flag, uint32_t epoch, const uint32_t* abort_word) {
  wait_flag_k<<<1, 1, 0, s>>>(flag, epoch, abort_word);
  check_launch("wait_flag");
  return 1;
}

int allreduce_scaled_peers(float* const* bufs, int D, int me, int64_t n, float scale, cudaStream_t s) {
  if (D < 1 || D > kMaxGroup) throw std::runtime_error("allreduce: 1 <= group size <= 32");
  if (n % 4) throw std::runtime_error("allreduce: length must be a multiple of 4");
  const int64_t n4 = n / 4, per = (n4 + D - 1) / D;
  const int64_t lo = std::min(n4, per * me), hi = std::min(n4, lo + per);
  if (hi <= lo) return 0;
  const int grid = static_cast<int>(std::min<int64_t>(4 * sm_count(), (hi - lo + 255) / 256));
  allreduce_scaled_k<<<grid, 256, 0, s>>>(bufs, D, lo, hi, scale);
  check_launch("allreduce_scaled_peers");
  return 1;
}

int xent_fwd_bwd(int dtype, void* logits, const int32_t* labels, float* loss, int T_, int V, float loss_scale,
                 float grad_scale, cudaStream_t s) {
  if (V % 8 == 0) {
    const int grid = (T_ + XR - 1) / XR;
    if (dtype == kBF16)
      xent_vec_k<bf16><<<grid, 256, 0, s>>>(static_cast<bf16*>(logits), labels, loss, T_, V, loss_scale, grad_scale);
    else
      xent_vec_k<float><<<grid, 256, 0, s>>>(static_cast<float*>(logits), labels, loss, T_, V, loss_scale,
                                             grad_scale);
  } else if (dtype == kBF16) {
    xent_k<bf16><<<T_, 256, 0, s>>>(static_cast<bf16*>(logits), labels, loss, V, loss_scale, grad_scale);
  } else {
    xent_k<float><<<T_, 256, 0, s>>>(static_cast<float*>(logits), labels, loss, V, loss_scale, grad_scale);
  }
  check_launch("xent");
  return 1;
}

int colsum_accum(int dtype, const void* dy, float* db, int T_, int n, int ld, cudaStream_t s) {
  if (n % 8 || ld % 8) throw std::runtime_error("colsum: columns and leading dimension must be multiples of 8");
  const int rows_per = 128;
  const dim3 grid((n + 255) / 256, (T_ + rows_per - 1) / rows_per);
  if (dtype == kBF16) colsum_k<bf16><<<grid, 256, 0, s>>>(static_cast<const bf16*>(dy), db, T_, n, ld, rows_per);
  else colsum_k<float><<<grid, 256, 0, s>>>(static_cast<const float*>(dy), db, T_, n, ld, rows_per);
  check_launch("colsum");
  return 1;
}

int optimizer_step(const OptimArgs& a, float* w, float* g, float* m, float* v, void* shadow, int64_t n,
                   cudaStream_t s) {
  const float bc1 = 1.f - std::pow(a.beta1, static_cast<float>(a.step));
  const float bc2 = 1.f - std::pow(a.beta2, static_cast<float>(a.step));
  optim_k<<<grid_for(n, 256), 256, 0, s>>>(a, w, g, m, v, static_cast<bf16*>(shadow), n, bc1, bc2);
  check_launch("optimizer");
  return 1;
}

int init_normal(float* p, int64_t n, float std, uint64_t seed, cudaStream_t s) {
  init_normal_k<<<grid_for(n, 256), 256, 0, s>>>(p, n, std, seed);
  check_launch("init_normal");
  return 1;
}

int fill_f32(float* p, int64_t n, float v, cudaStream_t s) {
  fill_k<<<grid_for(n, 256), 256, 0, s>>>(p, n, v);
  check_launch("fill");
  return 1;
}

int cast_f32_to_bf16(const float* src, void* dst, int64_t n, cudaStream_t s) {
  cast_k<<<grid_for(n, 256), 256, 0, s>>>(src, static_cast<bf16*>(dst), n);
  check_launch("cast");
  return 1;
}

}  // namespace wpk
