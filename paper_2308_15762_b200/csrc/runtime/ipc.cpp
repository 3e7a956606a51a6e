// CUDA-IPC transport of the runtime: one process per GPU, inter-stage
// messages pushed by copy engines over NVLink into the receiver's landing
// slots, with device-side signalling through stream memory operations.
//
// Reference semantics kept (src/simulate.cpp:117-155): a Send is buffered --
// it fires once its producer is done and never blocks the sender's compute
// stream; a Receive is *posted* at the start of the compute preceding its
// consumer (depth-1 prefetch, :123-133) and the bytes move at max(post,
// fire); the arrival gates only the consumer.  The incoming half of a
// BatchedExchange is posted the same way.  A send waits only on its producer
// and on its post, a compute only on its inputs -- the buffered replay of
// src/validate.cpp:438-495, hence deadlock-free.
//
// Memory: a landing slot is occupied from its post to the start of the
// consumer, which copies it into a stash buffer of the runtime's pool (the
// buffer the reference's memory_profile counts, src/analytics.cpp:61-76).
// Slots are assigned statically by walking each receiver's program (every
// rank derives every assignment, so a sender knows the slot address in its
// peer's arena) and reused as soon as the previous occupant was copied out:
// one or two slots per GPU instead of one per message.
//
// Layout of rank r's arena (one cudaMalloc, exported with cudaIpcGetMemHandle):
//   [ arrive[0..M) | posted[0..M) | ready[0..D) | done[0..D) ]  32-bit flags,
//       M = messages of the list, D = data-parallel replicas;
//       arrive[m] is used when r receives m, posted[m] when r sends m
//   [ landing slots of r ]
#include <algorithm>
#include <cstring>

#include "runtime/device_state.hpp"
#include "runtime/stream_ops.hpp"

namespace wprt {

using wavepipe::Action;

IpcPlan make_ipc_plan(const wavepipe::ActionList& list) {
  IpcPlan plan;
  const int P = list.config.devices;
  std::map<MsgKey, std::pair<int, int>> msgs;  // key -> (src, dst)
  std::map<int, std::vector<std::pair<int, int>>> groups;  // batch_group -> (device, position)
  for (int p = 0; p < P; ++p)
    for (int i = 0; i < static_cast<int>(list.per_device[p].size()); ++i) {
      const Action& a = list.per_device[p][i];
      if (a.kind == ActionKind::Send || a.kind == ActionKind::BatchedExchange) msgs[message_key(a)] = {p, a.peer};
      if (a.kind == ActionKind::BatchedExchange) groups[a.batch_group].push_back({p, i});
    }
  for (auto& [k, sd] : msgs) {
    plan.index[k] = static_cast<int>(plan.msgs.size());
    plan.msgs.push_back({sd.first, sd.second, -1});
  }
  // Landing-slot assignment per receiver, in its program order: message m is
  // posted at the start of the compute before the Receive (post index =
  // computes seen - 1) and copied out at the start of its consumer compute.
  // A slot is reusable by a post at compute c once its occupant was copied
  // out at a compute <= c (the copy-out is enqueued before c's start event).
  plan.slots.assign(P, 0);
  plan.issue_order.assign(P, {});
  for (int p = 0; p < P; ++p) {
    const auto& prog = list.per_device[p];
    std::map<MsgKey, int> consumer;  // input key -> compute index of its consumer
    for (int i = 0, c = 0; i < static_cast<int>(prog.size()); ++i)
      if (prog[i].is_compute()) consumer[input_key(prog[i])] = c++;
    std::vector<int> free_at;  // slot -> compute index of its last copy-out
    std::vector<std::pair<int, int>> by_consumer;  // (consumer compute, message)
    int computes = 0;
    auto assign = [&](const MsgKey& k) {
      const int m = plan.index.at(k), post = computes - 1;
      auto cit = consumer.find(k);
      if (cit == consumer.end()) throw wavepipe::SimulationError("IPC transport: received message has no consumer");
      const int consume = cit->second;
      int slot = -1;
      for (int s = 0; s < static_cast<int>(free_at.size()) && slot < 0; ++s)
        if (free_at[s] <= post) slot = s;
      if (slot < 0) {
        slot = static_cast<int>(free_at.size());
        free_at.push_back(consume);
      }
      free_at[slot] = consume;
      plan.msgs[m].slot = slot;
      by_consumer.push_back({consume, m});
    };
    for (int i = 0; i < static_cast<int>(prog.size()); ++i) {
      const Action& a = prog[i];
      if (a.is_compute()) {
        ++computes;
      } else if (a.kind == ActionKind::Receive) {
        assign(message_key(a));
      } else if (a.kind == ActionKind::BatchedExchange) {
        // the counterpart's outgoing message (ref include/wavepipe/action.hpp:67-73)
        for (const auto& [q, qi] : groups.at(a.batch_group))
          if (q != p) assign(message_key(list.per_device[q][qi]));
      }
    }
    plan.slots[p] = static_cast<int>(free_at.size());
    // Pushes to p go out in the order p consumes them.  A per-peer copy
    // stream is FIFO, so a push waits for every earlier one to that peer;
    // in consumer order those earlier messages are ones p needs before this
    // one anyway (each compute has one input), so the FIFO adds no wait the
    // list itself does not have and cannot deadlock a list the reference's
    // simulator runs (src/simulate.cpp:123-133).  Post order is not enough:
    // an exchange's incoming half can be posted early and consumed late
    // (Chimera), and a later-posted, earlier-consumed message would queue
    // behind it.
    std::sort(by_consumer.begin(), by_consumer.end());
    for (const auto& cm : by_consumer) plan.issue_order[p].push_back(cm.second);
  }
  for (const auto& m : plan.msgs)
    if (m.slot < 0) throw wavepipe::SimulationError("IPC transport: message without a receive");
  return plan;
}

void Runtime::ipc_setup() {
  const int P = list_.config.devices;
  const IpcPlan plan = make_ipc_plan(list_);
  ipc_index_ = plan.index;
  for (const auto& m : plan.msgs) ipc_msgs_.push_back(IpcMsg{m.src, m.dst, m.slot, 0});
  ipc_slots_ = plan.slots;
  for (int p = 0; p < P; ++p)
    for (int m : plan.issue_order[p])
      if (plan.msgs[m].src == rank_) ipc_send_order_[p].push_back(m);
  const size_t bytes = (message_bytes() + 255) & ~size_t(255);
  grad_group_.clear();
  for (int r = 0; r < replicas_; ++r) {
    grad_group_.push_back(grank(r, rank_));
    if (chimera_mirror() != rank_) grad_group_.push_back(grank(r, chimera_mirror()));
  }
  std::sort(grad_group_.begin(), grad_group_.end());
  group_me_ = static_cast<int>(std::find(grad_group_.begin(), grad_group_.end(), grank(replica_, rank_)) -
                               grad_group_.begin());
  grad_scale_ = 1.f / static_cast<float>(replicas_);
  const size_t G = grad_group_.size();
  // flags: arrive[M], posted[M], ready[G], done[G], then one probe word per global rank
  ipc_flag_bytes_ = ((2 * (ipc_msgs_.size() + G) + size_t(P) * replicas_) * sizeof(uint32_t) + 4095) & ~size_t(4095);
  for (IpcMsg& m : ipc_msgs_) m.data_off = ipc_flag_bytes_ + size_t(m.slot) * bytes;
  ipc_arena_bytes_ = ipc_flag_bytes_ + size_t(ipc_slots_[rank_]) * bytes;
  DeviceState& d = *devs_[0];
  DevGuard g(d.cuda);
  StreamOps::get();  // fail at creation, not mid-step, if the driver lacks stream memory ops
  ck(cudaMalloc(&ipc_arena_, ipc_arena_bytes_), "cudaMalloc IPC arena");
  // Abort word of the bounded waits: mapped pinned host memory the stall
  // watchdog sets from the host (no stream needed to release a wait).
  void* abort_mem = nullptr;
  ck(cudaHostAlloc(&abort_mem, sizeof(uint32_t), cudaHostAllocMapped), "cudaHostAlloc abort word");
  abort_host_ = static_cast<volatile uint32_t*>(abort_mem);
  *abort_host_ = 0;
  ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&abort_dev_), const_cast<uint32_t*>(abort_host_), 0),
     "abort word device pointer");
  ck(cudaMemset(ipc_arena_, 0, ipc_flag_bytes_), "memset IPC flags");
  ck(cudaDeviceSynchronize(), "IPC arena init");
  // One outgoing copy stream per peer this rank sends to; one signal stream.
  for (const IpcMsg& m : ipc_msgs_) {
    if (m.src == rank_ && !d.tx.count(m.dst)) {
      cudaStream_t s;
      ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
      d.tx[m.dst] = s;
    }
  }
  ck(cudaStreamCreateWithFlags(&d.sig, cudaStreamNonBlocking), "stream");
  ipc_peer_.assign(size_t(P) * replicas_, nullptr);
  dp_grads_.assign(G, nullptr);
  dp_grads_[group_me_] = d.grad;
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
  // The gradient group (same device in every other replica, Chimera mirror):
  // flags and gradients.
  for (int g = 0; g < static_cast<int>(grad_group_.size()); ++g) {
    if (g == group_me_) continue;
    const int q = grad_group_[g];
    if (!ipc_peer_[q]) ipc_peer_[q] = static_cast<char*>(open(q, 0));
    dp_grads_[g] = static_cast<float*>(open(q, 1));
  }
  if (grad_group_.size() > 1) {
    ck(cudaMalloc(&dp_grads_dev_, sizeof(float*) * grad_group_.size()), "cudaMalloc dp table");
    ck(cudaMemcpy(dp_grads_dev_, dp_grads_.data(), sizeof(float*) * grad_group_.size(), cudaMemcpyHostToDevice),
       "dp table");
  }
  ipc_connected_ = true;
  // Probe every mapped peer once with the operations the steps use -- a
  // copy-engine write and a stream-memory-op write into its arena (this
  // rank's own probe word) -- so an unsupported peer path fails here, at
  // set-up, where every rank can agree on a fallback, instead of mid-step.
  try {
    DeviceState& d = *devs_[0];
    const size_t probe =
        (2 * (ipc_msgs_.size() + grad_group_.size()) + size_t(grank(replica_, rank_))) * sizeof(uint32_t);
    for (char* peer : ipc_peer_) {
      if (!peer) continue;
      ck(cudaMemcpyAsync(peer + probe, ipc_arena_ + probe, sizeof(uint32_t), cudaMemcpyDeviceToDevice, d.sig),
         "IPC probe copy");
      StreamOps::write(d.sig, reinterpret_cast<uint32_t*>(peer + probe), 0u);
    }
    ck(cudaStreamSynchronize(d.sig), "IPC probe");
    ipc_ok_ = true;
  } catch (const std::exception& e) {
    ipc_ok_ = false;
    ipc_error_ = e.what();
    cudaGetLastError();
  }
}

void Runtime::ipc_release() {
  if (devs_.empty()) return;
  DevGuard g(devs_[0]->cuda);
  cudaDeviceSynchronize();
  for (char*& p : ipc_peer_) {
    if (p) cudaIpcCloseMemHandle(p);
    p = nullptr;
  }
  for (int g = 0; g < static_cast<int>(dp_grads_.size()); ++g)
    if (g != group_me_ && dp_grads_[g]) cudaIpcCloseMemHandle(dp_grads_[g]);
  dp_grads_.clear();
  if (dp_grads_dev_) cudaFree(dp_grads_dev_);
  dp_grads_dev_ = nullptr;
  if (ipc_arena_) cudaFree(ipc_arena_);
  ipc_arena_ = nullptr;
  if (abort_host_) cudaFreeHost(const_cast<uint32_t*>(abort_host_));
  abort_host_ = nullptr;
  if (devs_[0]->sig) cudaStreamDestroy(devs_[0]->sig);
  devs_[0]->sig = nullptr;
}

// Send / outgoing half of an exchange: the message is ready once its
// producer's event is recorded; it is issued (ipc_flush) in the receiver's
// consumer order.  Nothing here blocks the sender's compute stream.
void Runtime::ipc_send(DeviceState& d, const Action& a) {
  const MsgKey out = message_key(a);
  auto it = d.outbox.find(out);
  if (it == d.outbox.end()) throw wavepipe::SimulationError("runtime: send before its producer");
  const int m = ipc_index_.at(out);
  ipc_ready_[m] = {it->second, d.outbox_ready[out]};
  d.outbox.erase(it);
  d.outbox_ready.erase(out);
  ipc_flush(d, ipc_msgs_[m].dst);
}

// Issue every ready message to `peer` that is next in its consumer order: the
// per-peer copy stream waits for the producer (ready event) and for the
// receiver's post, pushes the bytes into the peer's landing slot, then raises
// the peer's arrival flag to this step's epoch.
void Runtime::ipc_flush(DeviceState& d, int peer_dev) {
  const auto& order = ipc_send_order_[peer_dev];
  size_t& next = ipc_send_next_[peer_dev];
  char* peer = ipc_peer_.at(grank(replica_, peer_dev));
  if (!peer) throw wavepipe::ConfigError("IPC peer not connected");
  cudaStream_t s = d.tx.at(peer_dev);
  while (next < order.size()) {
    const int m = order[next];
    auto it = ipc_ready_.find(m);
    if (it == ipc_ready_.end()) break;
    const IpcMsg& msg = ipc_msgs_[m];
    ck(cudaStreamWaitEvent(s, it->second.second, 0), "wait ready");
    launches_ += wpk::wait_flag(s, ipc_posted_flag(ipc_arena_, m), epoch_, abort_dev_);
    cudaEvent_t t0 = nullptr;
    if (tracing_) {
      t0 = next_event(d);
      ck(cudaEventRecord(t0, s), "record copy start");
    }
    ck(cudaMemcpyAsync(peer + msg.data_off, it->second.first->p, message_bytes(), cudaMemcpyDeviceToDevice, s),
       "IPC peer copy");
    if (tracing_) {
      cudaEvent_t t1 = next_event(d);
      ck(cudaEventRecord(t1, s), "record copy end");
      d.comm_recs.push_back({msg.src, msg.dst, t0, t1, &d, &d});
    }
    StreamOps::write(s, ipc_arrive_flag(peer, m), epoch_);
    d.pool->release(it->second.first, s);
    ipc_ready_.erase(it);
    ++next;
  }
}

// Receive / incoming half of an exchange: post it at the start of the compute
// before the consumer (the last start event; step begin if none), by writing
// the sender's posted flag from the signal stream; the consumer copies the
// slot out when it starts (ipc_land).
void Runtime::ipc_post(DeviceState& d, const MsgKey& k) {
  const int m = ipc_index_.at(k);
  const IpcMsg& msg = ipc_msgs_[m];
  char* peer = ipc_peer_.at(grank(replica_, msg.src));
  if (!peer) throw wavepipe::ConfigError("IPC peer not connected");
  ck(cudaStreamWaitEvent(d.sig, d.last_start ? d.last_start : d.step_begin, 0), "wait post point");
  StreamOps::write(d.sig, ipc_posted_flag(peer, m), epoch_);
  d.pending_ipc.push_back({k, m});
}

// At the start of compute `a` (compute stream): wait for its posted input to
// land, copy it out of the slot into a pool buffer (the stash entry), and
// hand that buffer to the compute.  The slot is free for the next post.
void Runtime::ipc_land(DeviceState& d, const Action& a) {
  const MsgKey want = input_key(a);
  for (size_t i = 0; i < d.pending_ipc.size(); ++i) {
    const auto [k, m] = d.pending_ipc[i];
    if (k.payload != want.payload || k.mb != want.mb || k.low != want.low) continue;
    const IpcMsg& msg = ipc_msgs_[m];
    launches_ += wpk::wait_flag(d.compute, ipc_arrive_flag(ipc_arena_, m), epoch_, abort_dev_);
    BufPtr b = d.pool->alloc(message_bytes(), d.compute, 0);
    ck(cudaMemcpyAsync(b->p, ipc_arena_ + msg.data_off, message_bytes(), cudaMemcpyDeviceToDevice, d.compute),
       "IPC slot copy-out");
    d.inbox[k] = b;
    d.pending_ipc.erase(d.pending_ipc.begin() + static_cast<long>(i));
    return;
  }
}

// Gradient all-reduce across this rank's gradient group (the D replicas of
// its pipeline device; for Chimera also their mirrors P-1-p, which hold the
// same stages for the opposite direction), on the compute stream right
// before the optimizer (the flush): publish "my grads are final" to every
// member, wait for theirs, run one peer-memory kernel in which each member
// sums its 1/G share over all G buffers (NVLink loads), scales by 1/D and
// writes the result back into all of them (NVLink stores), then publish /
// wait "done" so no buffer is reused while a peer still reads it.
void Runtime::dp_allreduce(DeviceState& d) {
  cudaStream_t s = d.compute;
  const int G = static_cast<int>(grad_group_.size());
  for (int g = 0; g < G; ++g)
    if (g != group_me_) StreamOps::write(s, ipc_dp_flag(ipc_peer_[grad_group_[g]], 0, group_me_), epoch_);
  for (int g = 0; g < G; ++g)
    if (g != group_me_) launches_ += wpk::wait_flag(s, ipc_dp_flag(ipc_arena_, 0, g), epoch_, abort_dev_);
  launches_ += wpk::allreduce_scaled_peers(dp_grads_dev_, G, group_me_, d.nparam, grad_scale_, s);
  for (int g = 0; g < G; ++g)
    if (g != group_me_) StreamOps::write(s, ipc_dp_flag(ipc_peer_[grad_group_[g]], 1, group_me_), epoch_);
  for (int g = 0; g < G; ++g)
    if (g != group_me_) launches_ += wpk::wait_flag(s, ipc_dp_flag(ipc_arena_, 1, g), epoch_, abort_dev_);
}

}  // namespace wprt
