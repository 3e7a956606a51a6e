// Private state of the GPU runtime shared by its translation units
// (executor.cpp: action interpreter and unit kernels; ipc.cpp: CUDA-IPC
// transport).  Not part of the public interface.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "capi_internal.hpp"
#include "runtime/runtime.hpp"

namespace wprt {

using wavepipe::ActionKind;

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw wpc::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

struct DevGuard {
  int prev = 0;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() { cudaSetDevice(prev); }
};

struct DeviceState {
  int pipe = 0;  // pipeline device (index into the ActionList)
  int cuda = 0;  // CUDA ordinal
  cudaStream_t compute = nullptr, copy = nullptr;
  std::unique_ptr<Pool> pool;
  std::vector<ParamSlot> params;
  std::unordered_map<std::string, int> by_name;
  int64_t nparam = 0;
  float *master = nullptr, *grad = nullptr, *m = nullptr, *v = nullptr;
  void* shadow = nullptr;  // bf16 copy of master (bf16 mode)
  float* loss = nullptr;
  int32_t *tokens = nullptr, *labels = nullptr;
  float* scores = nullptr;  // fp32 [mbs, heads, seq, seq] scratch (unfused attention)
  float* attn_delta = nullptr;  // fp32 [mbs, heads, seq] (fused attention backward)
  float* dq_acc = nullptr;      // fp32 [T, h]             (fused attention backward)
  float* ln_rows = nullptr;     // fp32 [T, 2]  LayerNorm-backward row sums (GEMM-fused path)
  int bwd_unit_lo = 0;          // first unit of the slice being run backward
  // Activation stash accounting (ref src/analytics.cpp:61-76): bytes held by
  // live (microbatch, slice) stash entries -- the slice's input message and
  // every tensor its units saved -- added when the forward is enqueued,
  // removed when its backward is; the high-water mark over all steps, and
  // per slice the largest entry seen.
  int64_t live_stash = 0, peak_stash = 0;
  uint64_t* clock_host = nullptr;  // mapped pinned word: %globaltimer at the traced step's begin
  uint64_t* clock_dev = nullptr;
  std::map<int, int64_t> slice_stash_bytes;
  bool dy_bias_done = false;    // the incoming dy's column sums are already in this unit's bias grad
  std::vector<std::pair<int, int>> be_partner;  // per position: (device, position) of a BE's counterpart

  // per-step program state
  size_t pc = 0;
  std::map<std::pair<int, int>, SliceStash> stash;
  std::map<MsgKey, BufPtr> handoff, inbox, outbox;
  std::map<MsgKey, cudaEvent_t> outbox_ready;
  std::vector<cudaEvent_t> pending;
  cudaEvent_t last_start = nullptr;
  cudaEvent_t step_begin = nullptr;
  std::vector<cudaEvent_t> events;
  size_t ev_next = 0;
  std::vector<uint8_t> published_at;  // BE positions whose outgoing message is published
  // IPC transport: per-peer outgoing copy streams.
  std::map<int, cudaStream_t> tx;
  // Start event of every compute enqueued this step (program position,
  // event): the watchdog names the first one that never started.
  std::vector<std::pair<size_t, cudaEvent_t>> starts;
  // IPC transport: messages whose landing slot the next compute copies out
  // (after its arrival flag reaches the step epoch), and the stream that
  // writes "posted" flags into senders' arenas.
  std::vector<std::pair<MsgKey, int>> pending_ipc;
  cudaStream_t sig = nullptr;

  struct Rec {
    int idx;
    ActionKind kind;
    int mb, slice;
    cudaEvent_t s, e;
  };
  struct CommRec {
    int src, dst;
    cudaEvent_t post, arrive;
    DeviceState* post_dev;
    DeviceState* arrive_dev;
  };
  std::vector<Rec> recs;
  std::vector<CommRec> comm_recs;
  struct GemmRec {
    double flops;
    cudaEvent_t s, e;
    std::string shape;
    bool attention = false;  // fused attention launch (reported apart from the GEMMs)
    bool hbm = false;        // HBM-bound kernel class (`shape` = class name, `flops` = bytes)
  };
  std::vector<GemmRec> gemm_recs;
};

}  // namespace wprt
