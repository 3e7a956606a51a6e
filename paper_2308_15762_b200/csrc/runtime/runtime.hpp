// GPU executor of a wavepipe ActionList.
//
// The reference executes lists only in abstract time (src/simulate.cpp:57-178);
// this runtime keeps that contract on real hardware:
//   Forward/Backward  kernels of the slice at local_module_rank on the device's
//                     compute stream; the stash slot of (microbatch, slice) lives
//                     from forward start to backward end (src/analytics.cpp:61-76)
//   Send              buffered: the producer's output is published with a ready
//                     event; nothing blocks the compute stream (:117-122)
//   Receive           the copy is *posted* at the start of the preceding compute
//                     (depth-1 prefetch, :123-133) and its arrival gates only the
//                     next compute
//   BatchedExchange   both directions of the pair move as one exchange; the
//                     incoming message is the counterpart's outgoing one (:134-155)
//   OptimizerStep     fused optimizer over the device's parameters (flush)
// Copies run on the *sender's* copy stream (push over NVLink / peer DMA, or
// D2D when several pipeline devices share one GPU), gated by the receiver's
// post event, so a message never lands before the receiver would have posted
// it -- the reference's memory bound holds.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "kernels/attention.cuh"
#include "kernels/gemm.cuh"
#include "kernels/ops.cuh"
#include "runtime/model.hpp"
#include "wavepipe/core.hpp"

namespace wprt {

// One device allocation from a per-device pool.  Message buffers (landing
// and outbox) carry an event recorded at free time so the next user on a
// different stream waits for the last one.
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  int pool_class = 0;  // 0 compute-only, 1 message
  cudaEvent_t ev = nullptr;
  bool ev_pending = false;
  cudaStream_t released_on = nullptr;
};
using BufPtr = std::shared_ptr<Buf>;

class Pool {
 public:
  Pool(int cuda_dev, cudaStream_t home) : dev_(cuda_dev), home_(home) {}
  ~Pool();
  BufPtr alloc(size_t bytes, cudaStream_t stream, int pool_class);
  void release(const BufPtr& b, cudaStream_t stream);
  size_t reserved() const { return reserved_; }
  void leak() { leak_ = true; }  // destructor skips cudaFree (streams blocked for good)

 private:
  int dev_;
  cudaStream_t home_;
  std::map<std::pair<int, size_t>, std::vector<BufPtr>> free_;
  std::vector<BufPtr> all_;
  size_t reserved_ = 0;
  bool leak_ = false;
};

// Saved tensors of one unit for its backward.
struct UnitStash {
  BufPtr x, ln, mean, rstd, a, b, c;  // attn: a=qkv b=P c=ctx; mlp: a=u b=g; head: a=dlogits
};

struct SliceStash {
  std::vector<UnitStash> units;  // in unit order of the slice
  int64_t bytes = 0;             // distinct stash buffers held (stash accounting)
};

struct MsgKey {
  int payload, mb, low;
  bool operator<(const MsgKey& o) const {
    return payload != o.payload ? payload < o.payload : mb != o.mb ? mb < o.mb : low < o.low;
  }
};

// Message identity (payload, microbatch, lower slice of the boundary), the
// reference's matching key (src/schedule.cpp:315-324, src/simulate.cpp:39-46).
inline MsgKey message_key(const wavepipe::Action& a) {
  const bool act = a.payload == static_cast<int>(wavepipe::Payload::Activation);
  const bool out = a.kind == wavepipe::ActionKind::Send || a.kind == wavepipe::ActionKind::BatchedExchange;
  return MsgKey{a.payload, a.microbatch,
                act ? (out ? a.slice_index : a.slice_index - 1) : (out ? a.slice_index - 1 : a.slice_index)};
}

// The message a compute consumes: Forward of slice s takes the activation
// of boundary s-1, Backward of slice s the gradient of boundary s.
inline MsgKey input_key(const wavepipe::Action& a) {
  return a.kind == wavepipe::ActionKind::Forward
             ? MsgKey{static_cast<int>(wavepipe::Payload::Activation), a.microbatch, a.slice_index - 1}
             : MsgKey{static_cast<int>(wavepipe::Payload::Gradient), a.microbatch, a.slice_index};
}

// Static plan of the CUDA-IPC transport, derived from the list alone (every
// rank computes the same one; no GPU needed -- tested on CPU): the global
// message table, each receiver's landing-slot assignment and push issue order.
struct IpcPlan {
  struct Msg {
    int src, dst, slot;
  };
  std::map<MsgKey, int> index;
  std::vector<Msg> msgs;
  std::vector<int> slots;                    // device -> landing slots it needs
  // device -> incoming message ids in the order of their consumer computes:
  // the order every sender issues its pushes to that device (see ipc.cpp)
  std::vector<std::vector<int>> issue_order;
};
IpcPlan make_ipc_plan(const wavepipe::ActionList& list);

struct Published {
  int src = -1;
  BufPtr buf;
  cudaEvent_t ready = nullptr;
};

struct ParamSlot {
  ParamDesc desc;
  int64_t offset = 0;  // element offset in the device's flat buffers
};

struct DeviceState;

class Runtime {
 public:
  Runtime(const wp_model_desc& desc, const wavepipe::ActionList& list, int transport, const int* device_ids,
          int rank);
  ~Runtime();

  // `producer`: the stream that wrote device-resident tokens/labels (nullptr:
  // the legacy default stream of their device); the step waits for it.
  float train_step(const int32_t* tokens, const int32_t* labels, bool on_device, cudaStream_t producer = nullptr);
  void set_stall_timeout(double seconds) { stall_timeout_s_ = seconds; }

  const wavepipe::SimTrace& trace() const { return trace_; }
  // %globaltimer (ns) on the (first local) device when the last traced step
  // began: trace times are relative to it, so adding it puts the ranks of
  // a job on one device clock.
  int64_t step_clock_ns() const { return step_clock_ns_; }
  void set_tracing(bool on) { tracing_ = on; }
  void set_update(bool on) { update_ = on; }
  // Per-GEMM CUDA events on the launching (compute) stream; accumulated over
  // the steps run while enabled: launches, executed FLOPs (2MNK per problem)
  // and summed kernel time.
  void set_profiling(bool on) { profiling_ = on; }
  void gemm_stats(int64_t* launches, double* flops, double* seconds) const {
    *launches = prof_launches_;
    *flops = prof_flops_;
    *seconds = prof_seconds_;
  }
  void attn_stats(int64_t* launches, double* flops, double* seconds) const {
    *launches = attn_launches_;
    *flops = attn_flops_;
    *seconds = attn_seconds_;
  }
  void reset_gemm_stats() {
    prof_launches_ = 0, prof_flops_ = 0, prof_seconds_ = 0;
    attn_launches_ = 0, attn_flops_ = 0, attn_seconds_ = 0;
    prof_shapes_.clear();
    hbm_stats_.clear();
  }
  // HBM-bound kernel classes timed while profiling: launches, algorithmic
  // bytes, seconds.
  int hbm_count() const { return static_cast<int>(hbm_stats_.size()); }
  void hbm_stat(int i, const char** name, int64_t* n, double* bytes, double* seconds) const {
    auto it = hbm_stats_.begin();
    std::advance(it, i);
    *name = it->first.c_str();
    *n = it->second.n;
    *bytes = it->second.flops;
    *seconds = it->second.seconds;
  }
  // Per GEMM shape: "MxNxK b<batch> <A,B majorness> c<causal>" -> (launches, flops, seconds).
  std::string gemm_report() const;
  int64_t launches() const { return launches_; }
  // Device memory of the local pipeline devices: stash/message pool and the
  // IPC landing slots (bytes).
  void memory(int64_t* pool_bytes, int64_t* landing_bytes) const;

  // Stash of pipeline device `pipe` (local): peak live bytes, and per slice
  // (index < nslices) the bytes of one (microbatch, slice) entry (0 if the
  // slice is not on that device).
  void stash_stats(int pipe, int64_t* peak_bytes, int64_t* slice_bytes, int nslices) const;
  int param_count() const { return static_cast<int>(param_index_.size()); }
  const ParamDesc& param_desc(int i, bool* owned) const;
  // IPC transport handshake: export this rank's landing arena (64-byte
  // cudaIpcMemHandle_t), then map every peer's from the handles of all ranks.
  void ipc_handle(void* out64) const;
  void ipc_connect(const void* handles, int nranks);
  // Result of the set-up probe of every mapped peer (copy + stream-op write).
  bool ipc_ok() const { return ipc_ok_; }
  const std::string& ipc_error() const { return ipc_error_; }
  // Bytes of one inter-stage message (activation or input-gradient).
  size_t message_bytes() const { return size_t(m_.tokens()) * m_.hidden * m_.act_bytes(); }
  void get_param(const std::string& name, float* host, int64_t n, bool grad);
  void set_param(const std::string& name, const float* host, int64_t n);

 private:
  struct ParamRef {
    int device;  // local device index owning it (-1: other process)
    int slot;
    ParamDesc desc;
  };

  void build_devices(const int* device_ids);
  void init_params(DeviceState& d);
  void enqueue_step();
  bool advance(DeviceState& d);
  void forward(DeviceState& d, const wavepipe::Action& a);
  void backward(DeviceState& d, const wavepipe::Action& a);
  void optimizer(DeviceState& d);
  void post_copy(DeviceState& dst, const MsgKey& key, Published msg);
  static int64_t stash_bytes(const SliceStash& st);
  void finish_step();          // watchdog-bounded wait for every local stream
  [[noreturn]] void stalled(); // diagnose, release this rank's device waits, throw
  BufPtr take_input(DeviceState& d, const MsgKey& key);
  void deliver(DeviceState& d, const MsgKey& key, BufPtr buf);
  cudaEvent_t next_event(DeviceState& d);
  void collect_trace();
  int owner_device(int mb, int slice) const;

  // unit kernels
  BufPtr unit_fwd(DeviceState& d, int unit, int mb, BufPtr x, UnitStash& st);
  BufPtr unit_bwd(DeviceState& d, int unit, int mb, UnitStash& st, BufPtr dy);
  void gemm(DeviceState& d, const wpk::GemmProblem& g);
  bool use_flash() const;  // fused tcgen05 attention (bf16, seq % 128 == 0, head_dim 64/128)
  wpk::AttnShape attn_shape() const;
  const void* weight(DeviceState& d, const std::string& name) const;  // act dtype (shadow or master)
  float* master(DeviceState& d, const std::string& name) const;
  float* grad(DeviceState& d, const std::string& name) const;

  ModelSpec m_;
  wavepipe::ActionList list_;
  std::vector<Unit> units_;
  std::vector<int> bounds_;  // slice -> unit range
  int transport_;
  int rank_;
  std::vector<std::unique_ptr<DeviceState>> devs_;  // local pipeline devices
  std::vector<int> dev_of_pipeline_;                // pipeline device -> index in devs_ (-1 remote)
  std::unordered_map<std::string, ParamRef> param_index_;
  std::vector<std::string> param_names_;
  std::map<MsgKey, Published> published_;
  bool tracing_ = false, update_ = true, profiling_ = false;
  int64_t prof_launches_ = 0, attn_launches_ = 0;
  double prof_flops_ = 0, prof_seconds_ = 0, attn_flops_ = 0, attn_seconds_ = 0;
  // Profiling of one fused-attention launch (fwd or bwd) on the compute stream.
  template <typename F>
  void timed_attention(DeviceState& d, bool backward, F&& launch);
  // Profiling of one HBM-bound kernel launch: class name, algorithmic bytes.
  template <typename F>
  void timed_hbm(DeviceState& d, const char* cls, double bytes, F&& launch);
  struct ShapeStat {
    int64_t n = 0;
    double flops = 0, seconds = 0;
  };
  std::map<std::string, ShapeStat> prof_shapes_;
  std::map<std::string, ShapeStat> hbm_stats_;  // flops field = bytes
  double stall_timeout_s_ = 300.0;
  int64_t step_clock_ns_ = 0;
  bool broken_ = false;    // a stalled step left the runtime unusable
  bool released_ = false;  // ... and its device waits were released (safe to free)
  cudaEvent_t input_ready_ = nullptr;
  int input_ready_dev_ = -1;
  int step_ = 0;
  int64_t launches_ = 0;
  wavepipe::SimTrace trace_;
  // CUDA-IPC transport (one process per GPU, copy-engine pushes over
  // NVLink); see ipc.cpp.  Every message m has a landing slot in its
  // receiver's arena (statically assigned from the receiver's program order,
  // reused as soon as the previous occupant was copied out) and two 32-bit
  // flags carrying the step epoch: posted[m] in the sender's arena (the
  // receiver reached the compute before the consumer, ref src/simulate.cpp:126)
  // and arrive[m] in the receiver's arena (the bytes landed).
  struct IpcMsg {
    int src, dst;
    int slot;         // landing slot in the receiver's arena
    size_t data_off;  // byte offset of that slot
  };
  std::vector<int> ipc_slots_;  // pipeline device -> landing slots of its arena
  // Sends to each peer are copied in the order that peer posts them (its
  // program order), so a copy waiting for its post never holds up a message
  // the peer needs first; the host defers a produced message until every
  // message the peer posts earlier has been issued.
  std::map<int, std::vector<int>> ipc_send_order_;  // peer -> message ids in the peer's consumer order
  std::map<int, size_t> ipc_send_next_;             // peer -> next position in that order
  std::map<int, std::pair<BufPtr, cudaEvent_t>> ipc_ready_;  // produced, not yet issued
  void ipc_flush(DeviceState& d, int peer);
  std::map<MsgKey, int> ipc_index_;
  std::vector<IpcMsg> ipc_msgs_;
  char* ipc_arena_ = nullptr;
  volatile uint32_t* abort_host_ = nullptr;  // stall release (mapped pinned host word)
  uint32_t* abort_dev_ = nullptr;            // its device address
  size_t ipc_flag_bytes_ = 0, ipc_arena_bytes_ = 0;
  std::vector<char*> ipc_peer_;  // global rank -> mapped arena (nullptr: not a peer)
  bool ipc_connected_ = false, ipc_ok_ = false;
  std::string ipc_error_;
  uint32_t epoch_ = 0;
  // Data-parallel replicas (list config D > 1, IPC transport only): global
  // rank = replica * P + pipeline device.  The arena's flag region also holds
  // ready[D] / done[D] for the gradient all-reduce of this pipeline device.
  int replicas_ = 1, replica_ = 0;
  // Gradient group of this rank: the global ranks whose gradient buffers are
  // reduced with its own at the OptimizerStep -- the same pipeline device in
  // every replica, plus, for Chimera, the mirrored device P-1-p that holds the
  // same two stages for the opposite direction.  Summed, then scaled by 1/D.
  std::vector<int> grad_group_;      // sorted global ranks (includes this rank)
  int group_me_ = 0;                 // this rank's index in grad_group_
  float grad_scale_ = 1.f;
  std::vector<float*> dp_grads_;     // group index -> that rank's grad buffer (mapped; own = local)
  float** dp_grads_dev_ = nullptr;   // same table in device memory (kernel argument)
  int grank(int replica, int pipe) const { return replica * list_.config.devices + pipe; }
  // Chimera places stage p (down) and P-1-p (up) on device p: devices p and
  // P-1-p hold the same two stages and sum their gradients.
  int chimera_mirror() const {
    return list_.config.scheme == wavepipe::Scheme::Chimera ? list_.config.devices - 1 - rank_ : rank_;
  }
  uint32_t* ipc_dp_flag(char* base, int which, int member) const {
    return reinterpret_cast<uint32_t*>(base) + 2 * ipc_msgs_.size() + which * grad_group_.size() + member;
  }
  void dp_allreduce(DeviceState& d);
  void ipc_setup();
  void ipc_release();
  uint32_t* ipc_arrive_flag(char* base, int m) const { return reinterpret_cast<uint32_t*>(base) + m; }
  uint32_t* ipc_posted_flag(char* base, int m) const {
    return reinterpret_cast<uint32_t*>(base) + ipc_msgs_.size() + m;
  }
  void ipc_send(DeviceState& d, const wavepipe::Action& a);
  void ipc_post(DeviceState& d, const MsgKey& k);
  void ipc_land(DeviceState& d, const wavepipe::Action& a);  // at a compute's start: its input
};

}  // namespace wprt
