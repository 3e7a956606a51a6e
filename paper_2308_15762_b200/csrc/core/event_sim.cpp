// Abstract-time executor: the semantic contract the GPU runtime implements.
//
// Same semantics as the reference simulator (src/simulate.cpp:57-178):
//   compute     occupies the engine from max(clock, pending arrival)     :93-111
//   optimizer   zero cost                                              :112-116
//   send        buffered; fires at the sender's engine-free time        :117-122
//   receive     posted at the start of the preceding compute (depth-1
//               prefetch); arrival = max(post, fire) + T_C gates only the
//               next compute                                           :123-133
//   batched ex. both sides reach it, then both engines are busy T_C     :134-155
//   stall       SimulationError naming the blocked action              :160-165
// Relaxation order does not affect any time (each is a max over its
// dependencies), and comm events are sorted at the end, so the trace is
// identical to the reference's.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <map>
#include <tuple>
#include <unordered_map>

#include "wavepipe/core.hpp"

namespace wavepipe {

namespace {

int64_t msg_key(const Action& a) {
  const bool act = a.payload == static_cast<int>(Payload::Activation);
  const bool out = a.kind == ActionKind::Send || a.kind == ActionKind::BatchedExchange;
  const int low = act ? (out ? a.slice_index : a.slice_index - 1)
                      : (out ? a.slice_index - 1 : a.slice_index);
  return (int64_t(a.payload & 3) << 60) | (int64_t(uint32_t(a.microbatch)) << 28) |
         int64_t(uint32_t(low + 1) & 0xFFFFFFF);
}

}  // namespace

SimTrace simulate(const ActionList& list, const CostModel& cost) {
  const ScheduleConfig& cfg = list.config;
  const int P = static_cast<int>(list.per_device.size());
  const double t_f = cost.slice_forward(cfg);
  const double t_b = cost.slice_backward(cfg);

  // batch_group -> its two (device, position) endpoints, checked up front.
  std::map<int, std::vector<std::pair<int, int>>> be;
  for (int d = 0; d < P; ++d) {
    const auto& st = list.per_device[d];
    for (int i = 0; i < static_cast<int>(st.size()); ++i) {
      if (st[i].kind == ActionKind::BatchedExchange) be[st[i].batch_group].emplace_back(d, i);
    }
  }
  for (const auto& [g, ends] : be) {
    if (ends.size() != 2 || ends[0].first == ends[1].first) {
      throw SimulationError("batch_group " + std::to_string(g) + " does not pair two devices");
    }
  }

  std::unordered_map<int64_t, double> fired;
  std::vector<std::vector<double>> reached(P);
  for (int d = 0; d < P; ++d) reached[d].assign(list.per_device[d].size(), -1.0);
  std::vector<std::vector<uint8_t>> has_reached(P);
  for (int d = 0; d < P; ++d) has_reached[d].assign(list.per_device[d].size(), 0);

  struct Dev {
    size_t pc = 0;
    double clock = 0.0, post = 0.0, gate = 0.0;
  };
  std::vector<Dev> dev(P);
  SimTrace tr;
  tr.intervals.resize(P);

  auto record = [&](int d, size_t pc, const Action& a, double s, double e) {
    TraceInterval iv;
    iv.action_index = static_cast<int>(pc);
    iv.kind = a.kind;
    iv.microbatch = a.microbatch;
    iv.slice_index = a.slice_index;
    iv.direction = microbatch_direction(cfg, a.microbatch);
    iv.start = s;
    iv.end = e;
    tr.intervals[d].push_back(iv);
  };

  for (bool moved = true; moved;) {
    moved = false;
    for (int d = 0; d < P; ++d) {
      Dev& v = dev[d];
      const auto& st = list.per_device[d];
      for (; v.pc < st.size(); ++v.pc, moved = true) {
        const Action& a = st[v.pc];
        if (a.is_compute()) {
          const double s = std::max(v.clock, v.gate);
          record(d, v.pc, a, s, s + (a.kind == ActionKind::Forward ? t_f : t_b));
          v.clock = s + (a.kind == ActionKind::Forward ? t_f : t_b);
          v.post = s;
          v.gate = 0.0;
        } else if (a.kind == ActionKind::OptimizerStep) {
          // free
        } else if (a.kind == ActionKind::Send) {
          fired[msg_key(a)] = v.clock;
        } else if (a.kind == ActionKind::Receive) {
          auto it = fired.find(msg_key(a));
          if (it == fired.end()) break;
          const double arrival = std::max(v.post, it->second) + cost.t_comm;
          v.gate = std::max(v.gate, arrival);
          tr.comm_events.push_back(CommEvent{a.peer, d, v.post, arrival});
        } else {  // BatchedExchange
          reached[d][v.pc] = v.clock;
          has_reached[d][v.pc] = 1;
          const auto& ends = be.at(a.batch_group);
          const auto other = ends[0] == std::make_pair(d, int(v.pc)) ? ends[1] : ends[0];
          if (!has_reached[other.first][other.second]) break;
          const double s = std::max(v.clock, reached[other.first][other.second]);
          const double e = s + cost.t_comm;
          record(d, v.pc, a, s, e);
          tr.comm_events.push_back(CommEvent{d, a.peer, s, e});
          v.clock = e;
        }
      }
    }
  }

  for (int d = 0; d < P; ++d) {
    if (dev[d].pc < list.per_device[d].size()) {
      throw SimulationError("simulation stalled: device " + std::to_string(d) + " blocked at " +
                            describe_action(list.per_device[d][dev[d].pc]));
    }
    tr.makespan = std::max(tr.makespan, dev[d].clock);
  }
  std::sort(tr.comm_events.begin(), tr.comm_events.end(), [](const CommEvent& x, const CommEvent& y) {
    return std::tie(x.arrival_time, x.post_time, x.src_device, x.dst_device) <
           std::tie(y.arrival_time, y.post_time, y.src_device, y.dst_device);
  });
  return tr;
}

namespace {

// Shortest round-trip decimal, with ".0" on integral values (JSON number).
std::string fmt_double(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, r.ptr);
  if (std::isfinite(v) && s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s;
}

}  // namespace

std::string trace_to_json(const SimTrace& tr) {
  std::string o = "{\n  \"makespan\": " + fmt_double(tr.makespan) + ",\n  \"intervals\": [";
  for (size_t d = 0; d < tr.intervals.size(); ++d) {
    o += d ? ",\n    [" : "\n    [";
    for (size_t i = 0; i < tr.intervals[d].size(); ++i) {
      const TraceInterval& iv = tr.intervals[d][i];
      o += i ? ",\n      {" : "\n      {";
      o += "\n        \"action_index\": " + std::to_string(iv.action_index);
      o += ",\n        \"kind\": \"" + std::string(action_kind_name(iv.kind)) + "\"";
      o += ",\n        \"microbatch\": " + std::to_string(iv.microbatch);
      o += ",\n        \"slice_index\": " + std::to_string(iv.slice_index);
      o += ",\n        \"direction\": \"" + std::string(direction_name(iv.direction)) + "\"";
      o += ",\n        \"start\": " + fmt_double(iv.start);
      o += ",\n        \"end\": " + fmt_double(iv.end) + "\n      }";
    }
    o += tr.intervals[d].empty() ? "]" : "\n    ]";
  }
  o += tr.intervals.empty() ? "],\n" : "\n  ],\n";
  o += "  \"comm_events\": [";
  for (size_t i = 0; i < tr.comm_events.size(); ++i) {
    const CommEvent& e = tr.comm_events[i];
    o += i ? ",\n    {" : "\n    {";
    o += "\n      \"src_device\": " + std::to_string(e.src_device);
    o += ",\n      \"dst_device\": " + std::to_string(e.dst_device);
    o += ",\n      \"post_time\": " + fmt_double(e.post_time);
    o += ",\n      \"arrival_time\": " + fmt_double(e.arrival_time) + "\n    }";
  }
  o += tr.comm_events.empty() ? "]\n}\n" : "\n  ]\n}\n";
  return o;
}

}  // namespace wavepipe
