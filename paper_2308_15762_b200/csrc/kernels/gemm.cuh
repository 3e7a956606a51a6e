// GEMM interface shared by the tensor-core (bf16, tcgen05) and SIMT (fp32
// parity mode) implementations.
//
//   C[z][m][n] (op)= sum_k A[z][m][k] * B[z][n][k]
//
// Each operand is row-major with a leading dimension; `mn_major` says which of
// its two logical indices is contiguous:
//   A: mn_major=false -> A[m][k] at ptr[m*ld + k]   (K-major, "row-major MxK")
//      mn_major=true  -> A[m][k] at ptr[k*ld + m]   (M-major, "row-major KxM")
//   B: mn_major=false -> B[n][k] at ptr[n*ld + k]   (K-major, torch Linear weight)
//      mn_major=true  -> B[n][k] at ptr[k*ld + n]   (N-major)
// so X @ W^T is (K,K), dY @ W is (K,N-major) and dY^T @ X is (M-major,N-major).
// A two-level batch index z = z1 + nb1*z2 adds z1*b1 + z2*b2 elements to every
// pointer (attention: z1 = head, z2 = sequence).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace wpk {

enum DType : int { kF32 = 0, kBF16 = 1 };

enum EpiMode : int {
  kEpiStore = 0,     // C = alpha*acc (+ bias[n])
  kEpiAccum = 1,     // C(f32) += alpha*acc              (gradient accumulation)
  kEpiResidual = 2,  // C = resid + alpha*acc + bias[n]   (block output)
  kEpiGelu = 3,      // aux = acc + bias (pre-activation), C = gelu(aux)
  kEpiDGelu = 4,     // C = acc * gelu'(aux)              (aux = pre-activation)
};

struct Operand {
  const void* ptr = nullptr;
  int64_t ld = 0;
  bool mn_major = false;
  int64_t b1 = 0, b2 = 0;  // batch strides (elements)
};

struct Epilogue {
  int mode = kEpiStore;
  float alpha = 1.0f;
  void* c = nullptr;  // dtype: c_dtype
  int c_dtype = kBF16;
  int64_t ldc = 0, c_b1 = 0, c_b2 = 0;
  const float* bias = nullptr;  // [N] fp32, optional
  const void* resid = nullptr;  // same dtype/ld as C (kEpiResidual)
  void* aux = nullptr;          // same dtype/ld as C (kEpiGelu out, kEpiDGelu in)
  // Optional: colsum[n] += sum over rows of the epilogue's output (fp32, the
  // bias gradient of the layer whose input gradient C is).  Fused into the
  // CTA-pair kernel's epilogue; other paths add a column-sum pass.
  float* colsum = nullptr;
  // Optional, CTA-pair kernel with a bf16 C only: LayerNorm-backward partials
  // of C = dLN for the LN whose input is ln_x (same dtype / ld as C):
  //   ln_dw[n] += sum_m C * xhat,   colsum (set it to ln_db) += sum_m C,
  //   ln_rows[2m] += sum_n C * ln_w[n],  ln_rows[2m+1] += sum_n C * ln_w[n] * xhat,
  // xhat = (ln_x - ln_mean[m]) * ln_rstd[m] -- the LN's dw / db and the two row
  // sums its dx needs, so dx becomes an elementwise pass (layernorm_bwd_dx_rows).
  const void* ln_x = nullptr;
  const float* ln_mean = nullptr;
  const float* ln_rstd = nullptr;
  const float* ln_w = nullptr;
  float* ln_dw = nullptr;
  float* ln_rows = nullptr;
  // Optional (store mode, bf16 C, CTA-pair TMA epilogue): per-row dot
  // products of C (rounded to bf16) with rd_x (same dtype / ld as C) over
  // column groups of rd_group, added into
  //   rd_out[((m / rd_seq) * (N / rd_group) + n / rd_group) * rd_seq + m % rd_seq]
  // -- attention's Delta = rowsum(dO * O) per (sequence, head, query) out of
  // the projection data-gradient GEMM that produces dO.
  const void* rd_x = nullptr;
  float* rd_out = nullptr;
  int rd_group = 0, rd_seq = 0;
};

// Causal structure inside each batch element (an s x s attention block,
// queries on M for kCausalSkipUpper / kCausalKUpToRow, keys on M for
// kCausalKFromRow).  Tiles / K blocks that only touch masked entries are not
// computed; the consumers never read those outputs.
enum CausalMode : int {
  kCausalNone = 0,
  kCausalSkipUpper = 1,  // C = Q K^T-like: skip output tiles entirely above the diagonal
  kCausalKUpToRow = 2,   // C = P V-like: K (keys) limited to <= the tile's last row
  kCausalKFromRow = 3,   // C = P^T dO-like: K (queries) starts at the tile's first row
};

struct GemmProblem {
  int M = 0, N = 0, K = 0;
  int nb1 = 1, nb2 = 1;
  int in_dtype = kBF16;  // A and B element type
  int causal = kCausalNone;
  Operand A, B;
  Epilogue epi;
};

// Launches on `stream`; returns the number of kernel launches issued (1).
// Throws std::runtime_error on an unsupported problem.  gemm() dispatches on
// in_dtype: bf16 -> gemm_tc (tcgen05), fp32 -> gemm_simt (FFMA parity mode).
int gemm(const GemmProblem& p, cudaStream_t stream);
int gemm_tc(const GemmProblem& p, cudaStream_t stream);
int gemm_simt(const GemmProblem& p, cudaStream_t stream);

#ifdef __CUDACC__
// GELU, tanh approximation (GPT-2), and its derivative; shared by epilogues
// and elementwise kernels so every path computes the same function.
__device__ __forceinline__ float gelu_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float u = k0 * (x + k1 * x * x * x);
  return 0.5f * x * (1.0f + tanhf(u));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float x2 = x * x;
  const float u = k0 * (x + k1 * x2 * x);
  const float t = tanhf(u);
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * k0 * (1.0f + 3.0f * k1 * x2);
}
#endif  // __CUDACC__

}  // namespace wpk
