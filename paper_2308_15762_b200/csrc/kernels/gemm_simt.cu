// fp32 GEMM on the FFMA pipes: the parity-mode path.  tcgen05 has no full
// fp32 kind (tf32 would miss the 1e-5 gate), so fp32 mode runs this tiled
// SIMT kernel with the same operand/epilogue contract as gemm_tc.
// 64x64 output tile per 256-thread CTA, 4x4 per thread, K step 16,
// double-buffered shared-memory tiles.
#include <cuda_bf16.h>

#include <stdexcept>

#include "kernels/gemm.cuh"
#include "kernels/ops.cuh"

namespace wpk {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

struct SimtParams {
  int M, N, K, nb1, causal;
  Operand A, B;
  Epilogue epi;
};

__device__ __forceinline__ float ld_op(const Operand& o, int64_t zoff, int r, int k) {
  const float* p = static_cast<const float*>(o.ptr) + zoff;
  return o.mn_major ? p[static_cast<int64_t>(k) * o.ld + r] : p[static_cast<int64_t>(r) * o.ld + k];
}

__global__ void __launch_bounds__(256) gemm_simt_kernel(const SimtParams p) {
  __shared__ float As[2][TK][TM + 4];
  __shared__ float Bs[2][TK][TN + 4];
  const int z = blockIdx.z;
  const int z1 = z % p.nb1, z2 = z / p.nb1;
  const int64_t za = z1 * p.A.b1 + z2 * p.A.b2;
  const int64_t zb = z1 * p.B.b1 + z2 * p.B.b2;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;

  // Causal K ranges on the 128-wide tiles the softmax writes (gemm.cuh).
  int k_lo = 0, k_hi = p.K;
  if (p.causal == kCausalKUpToRow) k_hi = min(p.K, ((m0 + TM - 1) / 128 + 1) * 128);
  if (p.causal == kCausalKFromRow) k_lo = (m0 / 128) * 128;

  // Each thread stages 4 A and 4 B elements per K step.
  auto stage = [&](int buf, int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * 256;  // 0..1023 over a 64 x 16 tile
      int r, k;
      if (p.A.mn_major) { r = e % TM; k = e / TM; } else { k = e % TK; r = e / TK; }
      const int gm = m0 + r, gk = k0 + k;
      As[buf][k][r] = (gm < p.M && gk < k_hi) ? ld_op(p.A, za, gm, gk) : 0.0f;
      if (p.B.mn_major) { r = e % TN; k = e / TN; } else { k = e % TK; r = e / TK; }
      const int gn = n0 + r;
      const int gk2 = k0 + k;
      Bs[buf][k][r] = (gn < p.N && gk2 < k_hi) ? ld_op(p.B, zb, gn, gk2) : 0.0f;
    }
  };

  float acc[4][4] = {};
  const int nk = (k_hi - k_lo + TK - 1) / TK;
  stage(0, k_lo);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) stage(cur ^ 1, k_lo + (kt + 1) * TK);
#pragma unroll
    for (int k = 0; k < TK; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[cur][k][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[cur][k][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

  const Epilogue& e = p.epi;
  const int64_t zc = z1 * e.c_b1 + z2 * e.c_b2;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= p.N) continue;
      const int64_t off = zc + static_cast<int64_t>(m) * e.ldc + n;
      float v = acc[i][j] * e.alpha;
      if (e.bias) v += e.bias[n];
      auto rd = [&](const void* q) {
        return e.c_dtype == kF32 ? static_cast<const float*>(q)[off]
                                 : __bfloat162float(static_cast<const __nv_bfloat16*>(q)[off]);
      };
      auto wr = [&](void* q, float x) {
        if (e.c_dtype == kF32) static_cast<float*>(q)[off] = x;
        else static_cast<__nv_bfloat16*>(q)[off] = __float2bfloat16_rn(x);
      };
      switch (e.mode) {
        case kEpiAccum:
          static_cast<float*>(e.c)[off] += v;
          break;
        case kEpiResidual:
          wr(e.c, v + rd(e.resid));
          break;
        case kEpiGelu: {
          const float pre = e.c_dtype == kF32 ? v : __bfloat162float(__float2bfloat16_rn(v));
          wr(e.aux, pre);
          wr(e.c, gelu_f(pre));
          break;
        }
        case kEpiDGelu:
          wr(e.c, v * gelu_grad_f(rd(e.aux)));
          break;
        default:
          wr(e.c, v);
      }
    }
  }
}

}  // namespace

int gemm_simt(const GemmProblem& g, cudaStream_t s) {
  if (g.in_dtype != kF32) throw std::runtime_error("gemm_simt: inputs must be fp32");
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return 0;
  SimtParams p{g.M, g.N, g.K, g.nb1, g.causal, g.A, g.B, g.epi};
  dim3 grid((g.N + TN - 1) / TN, (g.M + TM - 1) / TM, g.nb1 * g.nb2);
  gemm_simt_kernel<<<grid, 256, 0, s>>>(p);
  return 1;
}

int gemm(const GemmProblem& g, cudaStream_t s) {
  if (g.in_dtype == kBF16) return gemm_tc(g, s);
  int n = gemm_simt(g, s);
  if (g.epi.colsum) {
    if (g.nb1 * g.nb2 != 1) throw std::runtime_error("gemm: colsum needs an unbatched problem");
    n += colsum_accum(g.epi.c_dtype, g.epi.c, g.epi.colsum, g.M, g.N, static_cast<int>(g.epi.ldc), s);
  }
  return n;
}

}  // namespace wpk
