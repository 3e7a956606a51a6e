// Fused attention (flash-style) on tcgen05 for bf16 mode.
//
// Layout: qkv [T = mbs*seq, 3h] bf16 with Q, K, V of head j at columns
// j*D, h + j*D, 2h + j*D; ctx [T, h] bf16; lse [mbs, heads, seq] fp32 in the
// log2 domain (lse2 = max + log2(sum) of t = s * log2(e)/sqrt(D)).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace wpk {

struct AttnShape {
  int mbs, seq, heads, head_dim, hidden;  // hidden = heads * head_dim
  int causal;
};

// ctx = softmax(Q K^T / sqrt(D) [+ causal mask]) V per (sequence, head);
// also writes lse2.  Returns launches issued.
int flash_attn_fwd(const AttnShape& s, const void* qkv, void* ctx, float* lse2, cudaStream_t stream);

// Backward: dqkv[:, 0:h) = dQ, [h, 2h) = dK, [2h, 3h) = dV from qkv, the
// forward output `out` (ctx), its gradient `dout`, and lse2.  Scratch:
// delta [mbs, heads, seq] fp32, dq_acc [T, h] fp32.  Returns launches issued.
// dbias (optional, [3h] fp32): += the column sums of dQKV -- the QKV bias
// gradient -- from the fp32 dK / dV accumulators and dQ before rounding.
// delta_ready: Delta = rowsum(dO * O) [mbs, heads, seq] is already in `delta`
// (fused into the GEMM that produced dO); otherwise it is computed here.
int flash_attn_bwd(const AttnShape& s, const void* qkv, const void* out, const void* dout, const float* lse2,
                   float* delta, float* dq_acc, void* dqkv, cudaStream_t stream, float* dbias = nullptr,
                   bool delta_ready = false);

inline bool flash_supported(const AttnShape& s) {
  return s.seq % 128 == 0 && (s.head_dim == 64 || s.head_dim == 128);
}

}  // namespace wpk
