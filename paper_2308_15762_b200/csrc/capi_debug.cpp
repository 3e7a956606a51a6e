// Kernel-level entry points for the GPU tests (not part of the public
// wavepipe.h contract): run one GEMM problem synchronously on the current
// device so tests can compare each operand layout / epilogue against torch.
#include <cuda_runtime.h>

#include <string>

#include "capi_internal.hpp"
#include "kernels/gemm.cuh"

static int debug_gemm(int M, int N, int K, int nb1, int nb2, int in_dtype, const void* a, int64_t lda,
                             int a_mn, int64_t a_b1, int64_t a_b2, const void* b, int64_t ldb, int b_mn,
                             int64_t b_b1, int64_t b_b2, int mode, float alpha, void* c, int c_dtype, int64_t ldc,
                             int64_t c_b1, int64_t c_b2, const float* bias, const void* resid, void* aux,
                             int causal, float* colsum = nullptr) {
  try {
    wpk::GemmProblem g;
    g.M = M;
    g.N = N;
    g.K = K;
    g.nb1 = nb1;
    g.nb2 = nb2;
    g.in_dtype = in_dtype;
    g.causal = causal < 0 ? 0 : causal;
    g.A = wpk::Operand{a, lda, a_mn != 0, a_b1, a_b2};
    g.B = wpk::Operand{b, ldb, b_mn != 0, b_b1, b_b2};
    g.epi.mode = mode;
    g.epi.alpha = alpha;
    g.epi.c = c;
    g.epi.c_dtype = c_dtype;
    g.epi.ldc = ldc;
    g.epi.c_b1 = c_b1;
    g.epi.c_b2 = c_b2;
    g.epi.bias = bias;
    g.epi.resid = resid;
    g.epi.aux = aux;
    g.epi.colsum = colsum;
    wpk::gemm(g, nullptr);
    if (causal < 0) return WP_OK;  // async: the caller synchronises (timing)
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return wpc::fail(WP_ERR_CUDA, std::string("gemm: ") + cudaGetErrorString(e));
    return WP_OK;
  } catch (...) {
    return wpc::map_exception();
  }
}

extern "C" int wp_debug_gemm(int M, int N, int K, int nb1, int nb2, int in_dtype, const void* a, int64_t lda,
                             int a_mn, int64_t a_b1, int64_t a_b2, const void* b, int64_t ldb, int b_mn,
                             int64_t b_b1, int64_t b_b2, int mode, float alpha, void* c, int c_dtype, int64_t ldc,
                             int64_t c_b1, int64_t c_b2, const float* bias, const void* resid, void* aux) {
  return debug_gemm(M, N, K, nb1, nb2, in_dtype, a, lda, a_mn, a_b1, a_b2, b, ldb, b_mn, b_b1, b_b2, mode, alpha, c,
                    c_dtype, ldc, c_b1, c_b2, bias, resid, aux, 0);
}

// Same as wp_debug_gemm without the device synchronisation (back-to-back
// launches on the legacy stream for timing).
extern "C" int wp_debug_gemm_async(int M, int N, int K, int nb1, int nb2, int in_dtype, const void* a, int64_t lda,
                                   int a_mn, int64_t a_b1, int64_t a_b2, const void* b, int64_t ldb, int b_mn,
                                   int64_t b_b1, int64_t b_b2, int mode, float alpha, void* c, int c_dtype,
                                   int64_t ldc, int64_t c_b1, int64_t c_b2, const float* bias, const void* resid,
                                   void* aux) {
  return debug_gemm(M, N, K, nb1, nb2, in_dtype, a, lda, a_mn, a_b1, a_b2, b, ldb, b_mn, b_b1, b_b2, mode, alpha, c,
                    c_dtype, ldc, c_b1, c_b2, bias, resid, aux, -1);
}

// wp_debug_gemm plus the fused bias-gradient column sums (colsum[n] += sum of C's column n).
extern "C" int wp_debug_gemm_colsum(int M, int N, int K, int in_dtype, const void* a, int64_t lda, int a_mn,
                                    const void* b, int64_t ldb, int b_mn, int mode, void* c, int c_dtype,
                                    int64_t ldc, const void* aux, float* colsum) {
  return debug_gemm(M, N, K, 1, 1, in_dtype, a, lda, a_mn, 0, 0, b, ldb, b_mn, 0, 0, mode, 1.0f, c, c_dtype, ldc, 0,
                    0, nullptr, nullptr, const_cast<void*>(aux), 0, colsum);
}

extern "C" int wp_debug_gemm_causal(int M, int N, int K, int nb1, int nb2, int in_dtype, const void* a, int64_t lda,
                                    int a_mn, int64_t a_b1, int64_t a_b2, const void* b, int64_t ldb, int b_mn,
                                    int64_t b_b1, int64_t b_b2, int mode, float alpha, void* c, int c_dtype,
                                    int64_t ldc, int64_t c_b1, int64_t c_b2, const float* bias, const void* resid,
                                    void* aux, int causal) {
  return debug_gemm(M, N, K, nb1, nb2, in_dtype, a, lda, a_mn, a_b1, a_b2, b, ldb, b_mn, b_b1, b_b2, mode, alpha, c,
                    c_dtype, ldc, c_b1, c_b2, bias, resid, aux, causal);
}

#include "kernels/attention.cuh"

extern "C" int wp_debug_flash_fwd(int mbs, int seq, int heads, int head_dim, int causal, const void* qkv, void* ctx,
                                  float* lse2) {
  try {
    wpk::AttnShape s{mbs, seq, heads, head_dim, heads * head_dim, causal};
    wpk::flash_attn_fwd(s, qkv, ctx, lse2, nullptr);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return wpc::fail(WP_ERR_CUDA, std::string("flash fwd: ") + cudaGetErrorString(e));
    return WP_OK;
  } catch (...) {
    return wpc::map_exception();
  }
}

extern "C" int wp_debug_flash_bwd_bias(int mbs, int seq, int heads, int head_dim, int causal, const void* qkv,
                                       const void* out, const void* dout, const float* lse2, float* delta,
                                       float* dq_acc, void* dqkv, float* dbias);

extern "C" int wp_debug_flash_bwd(int mbs, int seq, int heads, int head_dim, int causal, const void* qkv,
                                  const void* out, const void* dout, const float* lse2, float* delta, float* dq_acc,
                                  void* dqkv) {
  return wp_debug_flash_bwd_bias(mbs, seq, heads, head_dim, causal, qkv, out, dout, lse2, delta, dq_acc, dqkv,
                                 nullptr);
}

// Same, also accumulating the QKV bias gradient (column sums of dQKV) into dbias.
extern "C" int wp_debug_flash_bwd_bias(int mbs, int seq, int heads, int head_dim, int causal, const void* qkv,
                                       const void* out, const void* dout, const float* lse2, float* delta,
                                       float* dq_acc, void* dqkv, float* dbias) {
  try {
    wpk::AttnShape s{mbs, seq, heads, head_dim, heads * head_dim, causal};
    wpk::flash_attn_bwd(s, qkv, out, dout, lse2, delta, dq_acc, dqkv, nullptr, dbias);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return wpc::fail(WP_ERR_CUDA, std::string("flash bwd: ") + cudaGetErrorString(e));
    return WP_OK;
  } catch (...) {
    return wpc::map_exception();
  }
}

#include "kernels/ops.cuh"

namespace {
int sync_status(const char* what) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return wpc::fail(WP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return WP_OK;
}
}  // namespace

extern "C" int wp_debug_layernorm(int dtype, int T, int h, const void* x, const float* w, const float* b, void* y,
                                  float* mean, float* rstd, const void* dy, const void* dres, void* dx, float* dw,
                                  float* db) {
  try {
    wpk::layernorm_fwd(dtype, x, w, b, y, mean, rstd, T, h, nullptr);
    if (dy) wpk::layernorm_bwd(dtype, dy, x, mean, rstd, w, dres, dx, dw, db, T, h, nullptr);
    return sync_status("layernorm");
  } catch (...) {
    return wpc::map_exception();
  }
}

extern "C" int wp_debug_xent(int dtype, void* logits, const int32_t* labels, float* loss, int T, int V,
                             float loss_scale, float grad_scale) {
  try {
    wpk::xent_fwd_bwd(dtype, logits, labels, loss, T, V, loss_scale, grad_scale, nullptr);
    return sync_status("xent");
  } catch (...) {
    return wpc::map_exception();
  }
}

#include "capi_internal.hpp"
#include "runtime/runtime.hpp"

// Host-only plan of the IPC transport for a list (no GPU): landing slots per
// device (`slots[devices]`), message count, and each message's
// (src, dst, slot) in `msgs[3 * n]` when non-null.  For CPU tests.
extern "C" int wp_debug_ipc_plan(const wp_list* list, int* slots, int* n_msgs, int* msgs, int capacity) {
  try {
    if (!list || !slots || !n_msgs) return wpc::fail(WP_ERR_CONFIG, "null argument");
    const wprt::IpcPlan plan = wprt::make_ipc_plan(list->list);
    for (size_t p = 0; p < plan.slots.size(); ++p) slots[p] = plan.slots[p];
    *n_msgs = static_cast<int>(plan.msgs.size());
    if (msgs)
      for (int i = 0; i < *n_msgs && i < capacity; ++i) {
        msgs[3 * i] = plan.msgs[i].src;
        msgs[3 * i + 1] = plan.msgs[i].dst;
        msgs[3 * i + 2] = plan.msgs[i].slot;
      }
    return WP_OK;
  } catch (...) {
    return wpc::map_exception();
  }
}

#include "runtime/model.hpp"

// The runtime's unit partition for a model and list (host only): bounds[S+1]
// and per-unit forward costs (costs[n_units], n_units returned), for CPU tests.
extern "C" int wp_debug_partition(const wp_model_desc* desc, const wp_list* list, int* bounds, double* costs,
                                  int* n_units) {
  try {
    if (!desc || !list || !bounds || !n_units) return wpc::fail(WP_ERR_CONFIG, "null argument");
    const auto m = wprt::ModelSpec::from_desc(*desc);
    const auto units = wprt::build_units(m);
    const auto& l = list->list;
    std::vector<int> slice_device(l.config.stages, 0);
    for (int d = 0; d < static_cast<int>(l.placement.assignment.size()); ++d)
      for (const auto& sl : l.placement.assignment[d]) slice_device[sl.index] = d;
    const auto b = wprt::partition_units(units, slice_device, l.config.devices);
    for (size_t i = 0; i < b.size(); ++i) bounds[i] = b[i];
    *n_units = static_cast<int>(units.size());
    if (costs)
      for (size_t i = 0; i < units.size(); ++i) costs[i] = units[i].cost;
    return WP_OK;
  } catch (...) {
    return wpc::map_exception();
  }
}
