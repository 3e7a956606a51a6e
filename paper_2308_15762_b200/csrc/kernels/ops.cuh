// HBM-bound kernels of the transformer stage (host-callable launchers).
// Activations are `act_t` = float (fp32 parity mode) or bf16; statistics,
// parameters, gradients and optimizer state are fp32.  Every launcher returns
// the number of kernel launches it issued, so the runtime can count them.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace wpk {

// x[t] = wte[tok[t]] + wpe[t % seq]          (tables in act dtype)
int embed_fwd(int dtype, const int32_t* tok, const void* wte, const void* wpe, void* x, int T, int seq, int h,
              cudaStream_t s);
// dwte[tok[t]] += dx[t]; dwpe[t % seq] += dx[t]   (fp32 grads, atomics)
int embed_bwd(int dtype, const int32_t* tok, const void* dx, float* dwte, float* dwpe, int T, int seq, int h,
              cudaStream_t s);

// y = (x - mean) * rstd * w + b; saves mean/rstd [T]
int layernorm_fwd(int dtype, const void* x, const float* w, const float* b, void* y, float* mean, float* rstd,
                  int T, int h, cudaStream_t s);
// dx = dres + LN'(dy); dw += sum dy*xhat; db += sum dy.  dres may be null.
int layernorm_bwd(int dtype, const void* dy, const void* x, const float* mean, const float* rstd, const float* w,
                  const void* dres, void* dx, float* dw, float* db, int T, int h, cudaStream_t s);

// dx of a LayerNorm backward whose dw / db and row sums were produced by the
// dgrad GEMM's epilogue (GemmProblem::epi.ln_*): rows[2t] = sum_n dy*w,
// rows[2t+1] = sum_n dy*w*xhat; dx = rstd (dy w - rows0/h - xhat rows1/h) + dres.
// dcol (optional, fp32 [h]): += the column sums of dx (the bf16-rounded
// values the next unit reads) -- the bias gradient of the unit below.
int layernorm_bwd_dx_rows(int dtype, const void* dy, const void* x, const float* mean, const float* rstd,
                          const float* w, const float* rows, const void* dres, void* dx, int T, int h, cudaStream_t s,
                          float* dcol = nullptr);

// Row softmax of fp32 scores S [rows, n] -> P (act dtype); causal masks
// column j > (row % n) (query position) and reads/writes only up to the end
// of the query's 128-wide tile.  Scale already applied to S.
int softmax_fwd(int dtype, const float* S, void* P, int rows, int n, int causal, cudaStream_t s);
// dS = scale * P * (dP - sum(dP*P)), written over P (act dtype).
int softmax_bwd(int dtype, const float* dP, void* P_inout, int rows, int n, float scale, int causal,
                cudaStream_t s);

// Fused cross-entropy: per row, loss += (lse - logit[label]) * loss_scale into
// *loss_accum (fp32 device scalar); logits overwritten with
// (softmax - onehot) * grad_scale.
int xent_fwd_bwd(int dtype, void* logits, const int32_t* labels, float* loss_accum, int T, int V, float loss_scale,
                 float grad_scale, cudaStream_t s);

// db[n] += sum_t dy[t][n]  (bias gradient)
int colsum_accum(int dtype, const void* dy, float* db, int T, int n, int ld, cudaStream_t s);

// Optimizer over a flat fp32 buffer; writes the act-dtype shadow (bf16 mode)
// and zeroes the gradient.  kind: 0 SGD, 1 AdamW (decoupled weight decay).
struct OptimArgs {
  int kind;
  float lr, beta1, beta2, eps, weight_decay;
  int step;  // 1-based, for bias correction
};
int optimizer_step(const OptimArgs& a, float* master, float* grad, float* m, float* v, void* shadow_bf16, int64_t n,
                   cudaStream_t s);

// Gradient all-reduce over peer memory: bufs[0..G) are the group's fp32
// gradient buffers (NVLink-mapped; bufs[me] local).  Member `me` owns
// elements [me*n/G, (me+1)*n/G) (float4 granules): it sums them over all G
// buffers, multiplies by `scale` (1/D for D data-parallel replicas) and
// stores the result into every buffer.
int allreduce_scaled_peers(float* const* bufs, int G, int me, int64_t n, float scale, cudaStream_t s);

// Bounded device-side wait of the IPC transport: the stream proceeds once
// *flag >= epoch (wrap-free, like CU_STREAM_WAIT_VALUE_GEQ) -- the flag
// written by a peer's stream memory op -- or once the host sets *abort
// (mapped pinned memory: the stall watchdog's release).  One thread; the
// acquire load at system scope orders the peer's bytes before what follows.
int wait_flag(cudaStream_t s, const uint32_t* flag, uint32_t epoch, const uint32_t* abort_word);

// *out = %globaltimer (ns) when the stream reaches this point: the common
// device clock that aligns the measured traces of the ranks of a job.
int stamp_globaltimer(uint64_t* out, cudaStream_t s);

// Deterministic N(0, std) init from a counter-based hash (Box-Muller).
int init_normal(float* p, int64_t n, float std, uint64_t seed, cudaStream_t s);
int fill_f32(float* p, int64_t n, float v, cudaStream_t s);
int cast_f32_to_bf16(const float* src, void* dst, int64_t n, cudaStream_t s);

}  // namespace wpk
