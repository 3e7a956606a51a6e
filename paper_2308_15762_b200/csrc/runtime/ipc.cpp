// CUDA-IPC transport of the runtime: one process per GPU, inter-stage
// messages pushed by copy engines over NVLink into the receiver's landing
// slots, with device-side signalling through stream memory operations.
//
// Reference semantics kept (src/simulate.cpp:117-155): a Send is buffered --
// it fires once its producer is done and never blocks the sender's compute
// stream; a Receive / the incoming half of a BatchedExchange gates only the
// next compute of the receiver.  The deadlock-freedom argument is the
// reference's buffered replay (src/validate.cpp:438-495): a send waits only
// on its producer and on the previous step's release of its own slot, a
// compute only on its own inputs.
//
// Layout of rank r's arena (one cudaMalloc, exported with cudaIpcGetMemHandle):
//   [ arrive[0..M) | free[0..M) | ready[0..D) | done[0..D) ]  32-bit flags,
//       M = messages of the list, D = data-parallel replicas
//   [ landing slot of every message whose receiver is r ]
// arrive[m] lives with the receiver (the sender's copy stream writes the
// epoch after the copy; the receiver's compute stream waits on it), free[m]
// lives with the sender (the receiver's stream writes the epoch when the
// slot is released, i.e. when the consuming slice's stash entry dies).
#include <cstring>

#include "runtime/device_state.hpp"
#include "runtime/stream_ops.hpp"

namespace wprt {

using wavepipe::Action;

void Runtime::ipc_setup() {
  // Global message table from the full list (identical on every rank).
  const int P = list_.config.devices;
  std::map<MsgKey, std::pair<int, int>> msgs;  // key -> (src, dst)
  for (int p = 0; p < P; ++p)
    for (const Action& a : list_.per_device[p])
      if (a.kind == ActionKind::Send || a.kind == ActionKind::BatchedExchange) msgs[message_key(a)] = {p, a.peer};
  const size_t bytes = (message_bytes() + 255) & ~size_t(255);
  ipc_flag_bytes_ = ((2 * (msgs.size() + replicas_) * sizeof(uint32_t)) + 4095) & ~size_t(4095);
  // Slot offsets inside every receiver's arena (each rank derives all of
  // them: a sender needs the offset in its peer's arena).
  std::vector<size_t> off(P, ipc_flag_bytes_);
  for (auto& [k, sd] : msgs) {
    ipc_index_[k] = static_cast<int>(ipc_msgs_.size());
    ipc_msgs_.push_back(IpcMsg{sd.first, sd.second, off[sd.second]});
    off[sd.second] += bytes;
  }
  ipc_arena_bytes_ = std::max<size_t>(off[rank_], 4096);
  DeviceState& d = *devs_[0];
  DevGuard g(d.cuda);
  StreamOps::get();  // fail at creation, not mid-step, if the driver lacks stream memory ops
  ck(cudaMalloc(&ipc_arena_, ipc_arena_bytes_), "cudaMalloc IPC arena");
  ck(cudaMemset(ipc_arena_, 0, ipc_flag_bytes_), "memset IPC flags");
  ck(cudaDeviceSynchronize(), "IPC arena init");
  // One outgoing copy stream per peer this rank sends to.
  for (const IpcMsg& m : ipc_msgs_) {
    if (m.src == rank_ && !d.tx.count(m.dst)) {
      cudaStream_t s;
      ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
      d.tx[m.dst] = s;
    }
  }
  ipc_peer_.assign(size_t(P) * replicas_, nullptr);
  dp_grads_.assign(replicas_, nullptr);
  dp_grads_[replica_] = d.grad;
}

void Runtime::ipc_handle(void* out64) const {
  if (transport_ != WP_TRANSPORT_IPC) throw wavepipe::ConfigError("runtime does not use the IPC transport");
  static_assert(2 * sizeof(cudaIpcMemHandle_t) == WP_IPC_HANDLE_BYTES, "IPC handle size");
  DevGuard g(devs_[0]->cuda);
  cudaIpcMemHandle_t h[2];
  ck(cudaIpcGetMemHandle(&h[0], ipc_arena_), "cudaIpcGetMemHandle (arena)");
  ck(cudaIpcGetMemHandle(&h[1], devs_[0]->grad), "cudaIpcGetMemHandle (grads)");
  std::memcpy(out64, h, sizeof(h));
}

void Runtime::ipc_connect(const void* handles, int nranks) {
  if (transport_ != WP_TRANSPORT_IPC) throw wavepipe::ConfigError("runtime does not use the IPC transport");
  if (nranks != list_.config.devices * replicas_) {
    throw wavepipe::ConfigError("ipc_connect: need one handle per rank (P * D)");
  }
  if (ipc_connected_) throw wavepipe::ConfigError("ipc_connect called twice");
  DevGuard g(devs_[0]->cuda);
  auto open = [&](int q, int which) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + size_t(q) * WP_IPC_HANDLE_BYTES + which * sizeof(h),
                sizeof(h));
    void* p = nullptr;
    ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    return p;
  };
  // Pipeline neighbours inside this replica.
  std::vector<uint8_t> peer(list_.config.devices, 0);
  for (const IpcMsg& m : ipc_msgs_) {
    if (m.src == rank_) peer[m.dst] = 1;
    if (m.dst == rank_) peer[m.src] = 1;
  }
  for (int q = 0; q < list_.config.devices; ++q)
    if (peer[q] && q != rank_) ipc_peer_[grank(replica_, q)] = static_cast<char*>(open(grank(replica_, q), 0));
  // The same pipeline device in every other replica: flags and gradients.
  for (int r = 0; r < replicas_; ++r) {
    if (r == replica_) continue;
    ipc_peer_[grank(r, rank_)] = static_cast<char*>(open(grank(r, rank_), 0));
    dp_grads_[r] = static_cast<float*>(open(grank(r, rank_), 1));
  }
  if (replicas_ > 1) {
    ck(cudaMalloc(&dp_grads_dev_, sizeof(float*) * replicas_), "cudaMalloc dp table");
    ck(cudaMemcpy(dp_grads_dev_, dp_grads_.data(), sizeof(float*) * replicas_, cudaMemcpyHostToDevice),
       "dp table");
  }
  ipc_connected_ = true;
}

void Runtime::ipc_release() {
  if (devs_.empty()) return;
  DevGuard g(devs_[0]->cuda);
  cudaDeviceSynchronize();
  for (char*& p : ipc_peer_) {
    if (p) cudaIpcCloseMemHandle(p);
    p = nullptr;
  }
  for (int r = 0; r < static_cast<int>(dp_grads_.size()); ++r)
    if (r != replica_ && dp_grads_[r]) cudaIpcCloseMemHandle(dp_grads_[r]);
  dp_grads_.clear();
  if (dp_grads_dev_) cudaFree(dp_grads_dev_);
  dp_grads_dev_ = nullptr;
  if (ipc_arena_) cudaFree(ipc_arena_);
  ipc_arena_ = nullptr;
}

// Send / outgoing half of an exchange: the per-peer copy stream waits for the
// producer (ready event) and for the receiver's release of this slot in the
// previous step, pushes the bytes into the peer's landing slot, then raises
// the peer's arrival flag to this step's epoch.
void Runtime::ipc_send(DeviceState& d, const Action& a) {
  const MsgKey out = message_key(a);
  auto it = d.outbox.find(out);
  if (it == d.outbox.end()) throw wavepipe::SimulationError("runtime: send before its producer");
  const int m = ipc_index_.at(out);
  const IpcMsg& msg = ipc_msgs_[m];
  char* peer = ipc_peer_.at(grank(replica_, msg.dst));
  if (!peer) throw wavepipe::ConfigError("IPC peer not connected");
  cudaStream_t s = d.tx.at(msg.dst);
  ck(cudaStreamWaitEvent(s, d.outbox_ready[out], 0), "wait ready");
  StreamOps::wait_geq(s, ipc_free_flag(ipc_arena_, m), epoch_ - 1);
  cudaEvent_t t0 = nullptr;
  if (tracing_) {
    t0 = next_event(d);
    ck(cudaEventRecord(t0, s), "record copy start");
  }
  ck(cudaMemcpyAsync(peer + msg.data_off, it->second->p, message_bytes(), cudaMemcpyDeviceToDevice, s),
     "IPC peer copy");
  if (tracing_) {
    cudaEvent_t t1 = next_event(d);
    ck(cudaEventRecord(t1, s), "record copy end");
    d.comm_recs.push_back({msg.src, msg.dst, t0, t1, &d, &d});
  }
  StreamOps::write(s, ipc_arrive_flag(peer, m), epoch_);
  d.pool->release(it->second, s);
  d.outbox.erase(it);
  d.outbox_ready.erase(out);
}

// Receive / incoming half of an exchange: the landing slot becomes the
// input buffer; the next compute waits for the arrival flag.
void Runtime::ipc_expect(DeviceState& d, const MsgKey& k) {
  const int m = ipc_index_.at(k);
  const IpcMsg& msg = ipc_msgs_[m];
  char* peer = ipc_peer_.at(grank(replica_, msg.src));
  if (!peer) throw wavepipe::ConfigError("IPC peer not connected");
  auto b = std::make_shared<Buf>();
  b->p = ipc_arena_ + msg.data_off;
  b->bytes = message_bytes();
  b->pool_class = 2;
  b->ipc_free_remote = ipc_free_flag(peer, m);
  b->ipc_epoch = epoch_;
  d.inbox[k] = b;
  d.pending_flags.push_back(ipc_arrive_flag(ipc_arena_, m));
}

// Gradient all-reduce across the D replicas of this pipeline device, on the
// compute stream right before the optimizer (the flush): publish "my grads
// are final" to every replica, wait for theirs, run one peer-memory kernel
// in which each replica averages its 1/D share over all D buffers (NVLink
// loads) and writes the mean back into all of them (NVLink stores), then
// publish / wait "done" so no buffer is reused while a peer still reads it.
void Runtime::dp_allreduce(DeviceState& d) {
  cudaStream_t s = d.compute;
  for (int r = 0; r < replicas_; ++r)
    if (r != replica_) StreamOps::write(s, ipc_dp_flag(ipc_peer_[grank(r, rank_)], 0, replica_), epoch_);
  for (int r = 0; r < replicas_; ++r)
    if (r != replica_) StreamOps::wait_geq(s, ipc_dp_flag(ipc_arena_, 0, r), epoch_);
  launches_ += wpk::allreduce_mean_peers(dp_grads_dev_, replicas_, replica_, d.nparam, s);
  for (int r = 0; r < replicas_; ++r)
    if (r != replica_) StreamOps::write(s, ipc_dp_flag(ipc_peer_[grank(r, rank_)], 1, replica_), epoch_);
  for (int r = 0; r < replicas_; ++r)
    if (r != replica_) StreamOps::wait_geq(s, ipc_dp_flag(ipc_arena_, 1, r), epoch_);
}

}  // namespace wprt
