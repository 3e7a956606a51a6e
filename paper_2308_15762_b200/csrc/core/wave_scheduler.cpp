// Deterministic greedy list scheduler + communication insertion.
//
// Produces per-device action streams that are bit-exact with the reference
// generator (src/schedule.cpp:475-499).  The reference rescans every
// (microbatch, slice) pair on every step -- O(P*B^2*S^2) -- but a microbatch's
// work is a single chain F0..F(S-1), B(S-1)..B0, so at any instant it has
// exactly one unscheduled node whose producer is done: its *frontier*.  We
// keep that frontier per microbatch and evaluate only those, O(B) per step.
// Because the selection rule is order-independent (a min over start times,
// ties to the lower device, then a strict total policy order), the incremental
// form yields the same stream as the full scan:
//   ready set        src/schedule.cpp:206-232
//   start / pick     src/schedule.cpp:235-252
//   arrival times    src/schedule.cpp:167-184   (produced + comm, same fp order)
//   admission        src/schedule.cpp:118-163   (wave cap <= P in flight :132-137)
//   policy           src/schedule.cpp:190-198   (bwd first, least remaining work,
//                                                 lower microbatch, traversal order)
//   counters         src/schedule.cpp:257-296
// insert_comm follows src/schedule.cpp:333-473 (Receive before the consumer,
// Send after the producer, adjacent mutual pairs fused into BatchedExchange,
// group ids in discovery order, trailing OptimizerStep).
#include <cstdint>
#include <limits>
#include <unordered_map>

#include "wavepipe/core.hpp"

namespace wavepipe {

namespace {

// Flattened owner table: for microbatch b, slice s -> (device, local rank),
// plus "first visit": no lower slice of b lives on the same device.
struct Chains {
  int B = 0, S = 0;
  std::vector<int> dev, rank;
  std::vector<uint8_t> first_visit;
  std::vector<uint8_t> dir;  // 0 down, 1 up

  int at(int b, int s) const { return b * S + s; }
};

Chains build_chains(const ScheduleConfig& cfg, const StagePlacement& pl) {
  Chains c;
  c.B = cfg.microbatches;
  c.S = cfg.stages;
  c.dev.resize(size_t(c.B) * c.S);
  c.rank.resize(c.dev.size());
  c.first_visit.resize(c.dev.size());
  c.dir.resize(c.B);
  for (int b = 0; b < c.B; ++b) {
    const Direction d = microbatch_direction(cfg, b);
    c.dir[b] = d == Direction::Down ? 0 : 1;
    // Chains of the same direction are identical; recompute cheaply anyway.
    for (int s = 0; s < c.S; ++s) {
      const SliceOwner o = slice_owner(cfg, pl, s, d);
      if (o.device < 0) throw ScheduleError("placement does not cover slice " + std::to_string(s));
      c.dev[c.at(b, s)] = o.device;
      c.rank[c.at(b, s)] = o.local_rank;
      bool first = true;
      for (int q = 0; q < s && first; ++q) first = c.dev[c.at(b, q)] != o.device;
      c.first_visit[c.at(b, s)] = first;
    }
  }
  return c;
}

struct Node {
  bool bwd = false;
  int mb = 0;
  int slice = 0;
};

class FrontierScheduler {
 public:
  FrontierScheduler(const ScheduleConfig& cfg, const Chains& ch, const CostModel& cost)
      : cfg_(cfg), ch_(ch), P_(cfg.devices), B_(cfg.microbatches), S_(cfg.stages),
        t_fwd_(cost.slice_forward(cfg)), t_bwd_(cost.slice_backward(cfg)), t_comm_(cost.t_comm) {
    fwd_end_.assign(size_t(B_) * S_, kNone);
    bwd_end_.assign(size_t(B_) * S_, kNone);
    next_fwd_.assign(B_, 0);
    next_bwd_.assign(B_, S_ - 1);
    engine_free_.assign(P_, 0.0);
    in_flight_.assign(size_t(P_) * 2, 0);
    fwd_done_.assign(P_, 0);
    fwd_total_.assign(P_, 0);
    for (size_t i = 0; i < ch_.dev.size(); ++i) ++fwd_total_[ch_.dev[i]];
    streams_.resize(P_);
  }

  std::vector<std::vector<Node>> run() {
    const long total = 2L * B_ * S_;
    std::vector<double> start(P_);
    std::vector<int> pick(P_);
    std::vector<double> arr(B_);
    std::vector<uint8_t> ok(B_);
    for (long step = 0; step < total; ++step) {
      // Pass 1: frontier nodes that are admissible, their arrival, and the
      // earliest feasible start per device.
      for (int d = 0; d < P_; ++d) start[d] = kInf;
      for (int b = 0; b < B_; ++b) {
        ok[b] = 0;
        const Node n = frontier(b);
        if (n.slice < 0) continue;
        const int d = ch_.dev[ch_.at(b, n.slice)];
        if (!admissible(n, d)) continue;
        ok[b] = 1;
        arr[b] = arrival(n);
        const double st = std::max(engine_free_[d], arr[b]);
        if (st < start[d]) start[d] = st;
      }
      // Pass 2: per device, the policy-best node among those runnable at its start.
      for (int d = 0; d < P_; ++d) pick[d] = -1;
      for (int b = 0; b < B_; ++b) {
        if (!ok[b]) continue;
        const Node n = frontier(b);
        const int d = ch_.dev[ch_.at(b, n.slice)];
        if (arr[b] > start[d]) continue;
        if (pick[d] < 0 || better(n, frontier(pick[d]))) pick[d] = b;
      }
      int best = -1;
      for (int d = 0; d < P_; ++d) {
        if (pick[d] >= 0 && (best < 0 || start[d] < start[best])) best = d;
      }
      if (best < 0) throw ScheduleError("schedule generation stalled with work remaining");
      commit(frontier(pick[best]), best, start[best]);
    }
    return streams_;
  }

 private:
  static constexpr double kNone = -1.0;
  static constexpr double kInf = std::numeric_limits<double>::infinity();

  Node frontier(int b) const {
    if (next_fwd_[b] < S_) return Node{false, b, next_fwd_[b]};
    return Node{true, b, next_bwd_[b]};  // slice -1 once finished
  }

  bool admissible(const Node& n, int d) const {
    const int i = ch_.at(n.mb, n.slice);
    const int dir = ch_.dir[n.mb];
    if (n.bwd) {
      return cfg_.scheme != Scheme::GPipe || fwd_done_[d] == fwd_total_[d];
    }
    switch (cfg_.scheme) {
      case Scheme::GPipe:
        return true;
      case Scheme::Dapple:
      case Scheme::Chimera: {
        const int pos = (cfg_.scheme == Scheme::Chimera && dir == 1) ? P_ - 1 - d : d;
        int dir_count = B_;
        if (cfg_.scheme == Scheme::Chimera) {
          const int down = (B_ + 1) / 2;
          dir_count = dir == 0 ? down : B_ - down;
        }
        const int cap = std::min(P_ - pos, dir_count);
        return in_flight_[d * 2 + dir] < cap || !ch_.first_visit[i];
      }
      case Scheme::Hanayo:
      case Scheme::ChimeraWave:
        return n.slice != 0 || entered_[dir] - exited_[dir] < P_;
    }
    return true;
  }

  double arrival(const Node& n) const {
    const int b = n.mb, s = n.slice;
    if (!n.bwd) {
      if (s == 0) return 0.0;
      const double produced = fwd_end_[ch_.at(b, s - 1)];
      const bool cross = ch_.dev[ch_.at(b, s - 1)] != ch_.dev[ch_.at(b, s)];
      return produced + (cross ? t_comm_ : 0.0);
    }
    if (s == S_ - 1) return fwd_end_[ch_.at(b, s)];  // loss turnaround, same device
    const double produced = bwd_end_[ch_.at(b, s + 1)];
    const bool cross = ch_.dev[ch_.at(b, s + 1)] != ch_.dev[ch_.at(b, s)];
    return produced + (cross ? t_comm_ : 0.0);
  }

  // Strict policy order (true if x runs before y).
  bool better(const Node& x, const Node& y) const {
    if (x.bwd != y.bwd) return x.bwd;
    const int rx = x.bwd ? x.slice : S_ - 1 - x.slice;
    const int ry = y.bwd ? y.slice : S_ - 1 - y.slice;
    if (rx != ry) return rx < ry;
    if (x.mb != y.mb) return x.mb < y.mb;
    if (x.slice != y.slice) return x.bwd ? x.slice > y.slice : x.slice < y.slice;
    return false;
  }

  void commit(const Node& n, int d, double st) {
    const double end = st + (n.bwd ? t_bwd_ : t_fwd_);
    engine_free_[d] = end;
    streams_[d].push_back(n);
    const int i = ch_.at(n.mb, n.slice);
    const int dir = ch_.dir[n.mb];
    if (!n.bwd) {
      fwd_end_[i] = end;
      ++next_fwd_[n.mb];
      ++fwd_done_[d];
      if (ch_.first_visit[i]) ++in_flight_[d * 2 + dir];
      if (n.slice == 0) ++entered_[dir];
    } else {
      bwd_end_[i] = end;
      --next_bwd_[n.mb];
      if (ch_.first_visit[i]) --in_flight_[d * 2 + dir];
      if (n.slice == 0) ++exited_[dir];
    }
  }

  const ScheduleConfig& cfg_;
  const Chains& ch_;
  const int P_, B_, S_;
  const double t_fwd_, t_bwd_, t_comm_;
  std::vector<double> fwd_end_, bwd_end_, engine_free_;
  std::vector<int> next_fwd_, next_bwd_;
  std::vector<int> in_flight_;  // [device][dir]: fwd_started - bwd_done
  std::vector<int> fwd_done_, fwd_total_;
  int entered_[2] = {0, 0}, exited_[2] = {0, 0};
  std::vector<std::vector<Node>> streams_;
};

// Message identity: (payload, microbatch, lower slice of the boundary), the
// key of src/schedule.cpp:315-324 and src/simulate.cpp:39-46.
int64_t message_key(const Action& a) {
  const bool act = a.payload == static_cast<int>(Payload::Activation);
  const bool out = a.kind == ActionKind::Send || a.kind == ActionKind::BatchedExchange;
  const int low = act ? (out ? a.slice_index : a.slice_index - 1)
                      : (out ? a.slice_index - 1 : a.slice_index);
  return (int64_t(a.payload) << 42) ^ (int64_t(uint32_t(a.microbatch)) << 21) ^
         int64_t(uint32_t(low + 1) & 0x1FFFFF);
}

}  // namespace

ActionList insert_comm(const ActionList& compute_only) {
  const ScheduleConfig& cfg = compute_only.config;
  const Chains ch = build_chains(cfg, compute_only.placement);
  const int P = cfg.devices, S = cfg.stages;

  // 1. Receive-before-consumer / Send-after-producer.
  std::vector<std::vector<Action>> streams(P);
  for (int d = 0; d < P; ++d) {
    auto& out = streams[d];
    for (const Action& c : compute_only.per_device[d]) {
      if (!c.is_compute()) throw ScheduleError("insert_comm expects compute-only input streams");
      const bool bwd = c.kind == ActionKind::Backward;
      const int s = c.slice_index;
      const int payload = static_cast<int>(bwd ? Payload::Gradient : Payload::Activation);
      auto comm = [&](ActionKind k, int other) {
        Action a;
        a.kind = k;
        a.microbatch = c.microbatch;
        a.slice_index = s;
        a.local_module_rank = ch.rank[ch.at(c.microbatch, s)];
        a.peer = ch.dev[ch.at(c.microbatch, other)];
        a.payload = payload;
        out.push_back(a);
      };
      const int src = bwd ? s + 1 : s - 1;
      const int dst = bwd ? s - 1 : s + 1;
      if (src >= 0 && src < S && ch.dev[ch.at(c.microbatch, src)] != d) comm(ActionKind::Receive, src);
      out.push_back(c);
      if (dst >= 0 && dst < S && ch.dev[ch.at(c.microbatch, dst)] != d) comm(ActionKind::Send, dst);
    }
  }

  // 2. Where each message is sent / received.
  struct Ref { int dev, pos; };
  std::unordered_map<int64_t, Ref> send_at, recv_at;
  for (int d = 0; d < P; ++d) {
    for (int i = 0; i < static_cast<int>(streams[d].size()); ++i) {
      const Action& a = streams[d][i];
      if (a.kind == ActionKind::Send) send_at[message_key(a)] = Ref{d, i};
      if (a.kind == ActionKind::Receive) recv_at[message_key(a)] = Ref{d, i};
    }
  }
  auto find = [](const std::unordered_map<int64_t, Ref>& m, int64_t k) {
    auto it = m.find(k);
    if (it == m.end()) throw ScheduleError("insert_comm: unmatched message");
    return it->second;
  };

  // 3. Greedy left-to-right fusion of mutually adjacent opposing pairs.
  std::vector<std::vector<int>> group(P);
  for (int d = 0; d < P; ++d) group[d].assign(streams[d].size(), -1);
  int next_group = 0;
  for (int d = 0; d < P; ++d) {
    const auto& st = streams[d];
    for (int i = 0; i + 1 < static_cast<int>(st.size()); ++i) {
      if (group[d][i] >= 0 || group[d][i + 1] >= 0) continue;
      const Action& x = st[i];
      const Action& y = st[i + 1];
      const bool opposing = (x.kind == ActionKind::Send && y.kind == ActionKind::Receive) ||
                            (x.kind == ActionKind::Receive && y.kind == ActionKind::Send);
      if (!opposing || x.peer != y.peer || x.peer < 0) continue;
      const Action& snd = x.kind == ActionKind::Send ? x : y;
      const Action& rcv = x.kind == ActionKind::Send ? y : x;
      // Message key of a Receive keyed as the peer's Send and vice versa.
      const Ref their_recv = find(recv_at, message_key(snd));
      const Ref their_send = find(send_at, message_key(rcv));
      const int q = x.peer;
      if (their_recv.dev != q || their_send.dev != q) continue;
      if (std::abs(their_recv.pos - their_send.pos) != 1) continue;
      if (group[q][their_recv.pos] >= 0 || group[q][their_send.pos] >= 0) continue;
      const int g = next_group++;
      group[d][i] = group[d][i + 1] = g;
      group[q][their_recv.pos] = group[q][their_send.pos] = g;
    }
  }

  // 4. Collapse fused pairs (the BE carries the outgoing message, at the
  //    pair's first position) and append the flush.
  ActionList out;
  out.config = cfg;
  out.placement = compute_only.placement;
  out.per_device.resize(P);
  for (int d = 0; d < P; ++d) {
    const auto& st = streams[d];
    auto& dst = out.per_device[d];
    dst.reserve(st.size() + 1);
    for (size_t i = 0; i < st.size(); ++i) {
      if (group[d][i] < 0) {
        dst.push_back(st[i]);
        continue;
      }
      Action be = st[i].kind == ActionKind::Send ? st[i] : st[i + 1];
      be.kind = ActionKind::BatchedExchange;
      be.batch_group = group[d][i];
      dst.push_back(be);
      ++i;
    }
    Action opt;
    opt.kind = ActionKind::OptimizerStep;
    dst.push_back(opt);
  }
  return out;
}

ActionList generate_schedule(const StagePlacement& placement, const ScheduleConfig& cfg,
                             const CostModel& cost) {
  if (placement.device_count() != cfg.devices) {
    throw ScheduleError("placement device count does not match config");
  }
  const Chains ch = build_chains(cfg, placement);
  FrontierScheduler sched(cfg, ch, cost);
  const auto streams = sched.run();
  ActionList compute;
  compute.config = cfg;
  compute.placement = placement;
  compute.per_device.resize(cfg.devices);
  for (int d = 0; d < cfg.devices; ++d) {
    for (const Node& n : streams[d]) {
      Action a;
      a.kind = n.bwd ? ActionKind::Backward : ActionKind::Forward;
      a.microbatch = n.mb;
      a.slice_index = n.slice;
      a.local_module_rank = ch.rank[ch.at(n.mb, n.slice)];
      compute.per_device[d].push_back(a);
    }
  }
  return insert_comm(compute);
}

}  // namespace wavepipe
