// Trace analytics: bubble ratio, activation-stash bound, Hanayo Eq. 1.
//
//   bubble_ratio              src/analytics.cpp:32-46  (F/B busy only; BE is bubble;
//                                                       same summation order)
//   memory_profile            src/analytics.cpp:48-91  (+frac at fwd start,
//                                                       -frac at bwd end, frees first)
//   activation_variance       src/analytics.cpp:93-105
//   zone_bubbles              src/analytics.cpp:107-122
//   analytic_bubble_hanayo    src/analytics.cpp:124-157 (Eq. 1)
//   analytic_bubble_simplified src/analytics.cpp:159-164
//   compute_metrics           src/analytics.cpp:171-186
#include <algorithm>
#include <charconv>
#include <iomanip>
#include <sstream>
#include <unordered_map>

#include "wavepipe/core.hpp"

namespace wavepipe {

double bubble_ratio(const SimTrace& tr) {
  if (tr.makespan <= 0.0) {
    throw std::invalid_argument("bubble ratio undefined for a zero-makespan trace");
  }
  double busy = 0.0;
  for (const auto& dev : tr.intervals) {
    for (const TraceInterval& iv : dev) {
      if (iv.kind == ActionKind::Forward || iv.kind == ActionKind::Backward) busy += iv.end - iv.start;
    }
  }
  return 1.0 - busy / (static_cast<double>(tr.intervals.size()) * tr.makespan);
}

MemoryProfile memory_profile(const SimTrace& tr, const ActionList& list) {
  const int P = static_cast<int>(list.per_device.size());
  MemoryProfile mp;
  mp.weight_units.assign(P, Rational(0));
  mp.peak_activation_units.assign(P, Rational(0));
  for (int d = 0; d < P; ++d) {
    std::unordered_map<int, Rational> share;
    for (const StageSlice& sl : list.placement.assignment[d]) {
      mp.weight_units[d] += sl.fraction;
      share[sl.index] = sl.fraction;
    }
    std::vector<std::pair<double, Rational>> ev;
    for (const TraceInterval& iv : tr.intervals[d]) {
      if (iv.kind == ActionKind::BatchedExchange) continue;
      auto it = share.find(iv.slice_index);
      if (it == share.end()) {
        throw std::invalid_argument("trace interval references slice " +
                                    std::to_string(iv.slice_index) + " not placed on device " +
                                    std::to_string(d));
      }
      if (iv.kind == ActionKind::Forward) ev.emplace_back(iv.start, it->second);
      else ev.emplace_back(iv.end, -it->second);
    }
    std::sort(ev.begin(), ev.end(), [](const auto& x, const auto& y) {
      return x.first != y.first ? x.first < y.first : x.second < y.second;
    });
    Rational live(0), peak(0);
    for (const auto& e : ev) {
      live += e.second;
      if (peak < live) peak = live;
    }
    mp.peak_activation_units[d] = peak;
  }
  return mp;
}

Rational activation_variance(const MemoryProfile& mp) {
  const auto& x = mp.peak_activation_units;
  if (x.empty()) return Rational(0);
  Rational mean(0);
  for (const Rational& v : x) mean += v;
  mean /= Rational(static_cast<int64_t>(x.size()));
  Rational acc(0);
  for (const Rational& v : x) acc += (v - mean) * (v - mean);
  return acc / Rational(static_cast<int64_t>(x.size()));
}

ZoneBubbles zone_bubbles(const ZoneBubbleInput& in) {
  if (in.devices < 1) throw ConfigError("zone bubbles: P must be >= 1");
  if (in.waves < 1) throw ConfigError("zone bubbles: W must be >= 1");
  if (in.local_rank < 0 || in.local_rank >= in.devices) throw ConfigError("zone bubbles: LR must be in [0, P)");
  const double two_w = 2.0 * in.waves;
  ZoneBubbles z;
  z.a = in.t_forward / two_w + in.t_comm;
  z.b = (static_cast<double>(in.devices - in.local_rank) / two_w) * (in.t_backward - in.t_forward) +
        2.0 * in.t_comm;
  z.c_first = in.t_backward + 2.0 * in.t_comm;
  z.c_second = in.t_backward + in.t_comm;
  return z;
}

Rational analytic_bubble_hanayo(int P, int W, const Rational& tf, const Rational& tb,
                                const Rational& tc) {
  if (P < 2) throw ConfigError("analytic bubble ratio requires P >= 2");
  if (W < 1) throw ConfigError("analytic bubble ratio requires W >= 1");
  const int64_t p = P, w = W;
  // Eq. 1:  [T_B/W + (1 + 2W + 2/P + (P-2)/3) T_C]
  //       / [P/(P-1) T_F + (1/(2W) + P/(P-1)) T_B + ((P-2)/2 + 4W) T_C]
  const Rational top = tb / Rational(w) +
                       (Rational(1) + Rational(2 * w) + Rational(2, p) + Rational(p - 2, 3)) * tc;
  const Rational bot = Rational(p, p - 1) * tf + (Rational(1, 2 * w) + Rational(p, p - 1)) * tb +
                       (Rational(p - 2, 2) + Rational(4 * w)) * tc;
  if (bot == Rational(0)) throw ConfigError("analytic bubble ratio undefined for an all-zero cost model");
  return top / bot;
}

double analytic_bubble_hanayo_d(int P, int W, double tf, double tb, double tc) {
  if (P < 2) throw ConfigError("analytic bubble ratio requires P >= 2");
  if (W < 1) throw ConfigError("analytic bubble ratio requires W >= 1");
  const double p = P, w = W;
  const double top = tb / w + (1.0 + 2.0 * w + 2.0 / p + (p - 2.0) / 3.0) * tc;
  const double bot = (p / (p - 1.0)) * tf + (1.0 / (2.0 * w) + p / (p - 1.0)) * tb +
                     ((p - 2.0) / 2.0 + 4.0 * w) * tc;
  if (bot == 0.0) throw ConfigError("analytic bubble ratio undefined for an all-zero cost model");
  return top / bot;
}

Rational analytic_bubble_simplified(int P, int W) {
  if (P < 2) throw ConfigError("simplified bubble ratio requires P >= 2");
  if (W < 1) throw ConfigError("simplified bubble ratio requires W >= 1");
  const int64_t p = P, w = W;
  return Rational(2 * p - 2, 3 * p * w + p - 1);
}

double analytic_chimera_k(int P) {
  const double p = P;
  return p * p / 2.0 - p;
}

MetricsReport compute_metrics(const SimTrace& tr, const ActionList& list) {
  MetricsReport r;
  r.makespan = tr.makespan;
  r.bubble_ratio = bubble_ratio(tr);
  r.busy.assign(tr.intervals.size(), 0.0);
  for (size_t d = 0; d < tr.intervals.size(); ++d) {
    for (const TraceInterval& iv : tr.intervals[d]) {
      if (iv.kind == ActionKind::Forward || iv.kind == ActionKind::Backward) r.busy[d] += iv.end - iv.start;
    }
  }
  r.memory = memory_profile(tr, list);
  r.activation_variance = activation_variance(r.memory);
  return r;
}

std::string metrics_to_text(const MetricsReport& r) {
  std::ostringstream os;
  os << "makespan:            " << r.makespan << "\n"
     << "bubble_ratio:        " << r.bubble_ratio << "\n"
     << "activation_variance: " << r.activation_variance.to_string() << "\n"
     << "device  busy  weight_units  peak_activation_units\n";
  for (size_t d = 0; d < r.busy.size(); ++d) {
    os << std::left << std::setw(8) << d << std::setw(6) << r.busy[d] << std::setw(14)
       << r.memory.weight_units[d].to_string() << r.memory.peak_activation_units[d].to_string()
       << "\n";
  }
  return os.str();
}

std::string metrics_to_json(const MetricsReport& r) {
  auto num = [](double v) {
    char b[64];
    auto e = std::to_chars(b, b + sizeof b, v);
    std::string s(b, e.ptr);
    if (s.find_first_of(".eE") == std::string::npos) s += ".0";
    return s;
  };
  std::string o = "{\n  \"makespan\": " + num(r.makespan) + ",\n  \"bubble_ratio\": " +
                  num(r.bubble_ratio) + ",\n  \"activation_variance\": \"" +
                  r.activation_variance.to_string() + "\",\n  \"devices\": [";
  for (size_t d = 0; d < r.busy.size(); ++d) {
    o += d ? ",\n    {" : "\n    {";
    o += "\n      \"device\": " + std::to_string(d) + ",\n      \"busy\": " + num(r.busy[d]) +
         ",\n      \"weight_units\": \"" + r.memory.weight_units[d].to_string() +
         "\",\n      \"peak_activation_units\": \"" +
         r.memory.peak_activation_units[d].to_string() + "\"\n    }";
  }
  o += r.busy.empty() ? "]\n}\n" : "\n  ]\n}\n";
  return o;
}

}  // namespace wavepipe
