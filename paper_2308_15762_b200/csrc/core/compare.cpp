// Scheme comparison (ref src/analytics.cpp:221-331): generate, simulate and
// measure each requested scheme at a shared device budget, in throughput
// order.  The same rows feed the GPU runtime's measured comparison
// (bench.py --compare): there each row's makespan is a measured step.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cmath>
#include <sstream>

#include "wavepipe/core.hpp"

namespace wavepipe {

namespace {

// One row's schedule config and cost: chimera-wave is evaluated as one of its
// two symmetric device groups (ref src/analytics.cpp:236-247).
ScheduleConfig row_config(const CompareRequest& req, int budget, int microbatches, const CostModel& base,
                          CostModel* cost) {
  *cost = base;
  if (req.scheme != Scheme::ChimeraWave) return make_config(req.scheme, budget, microbatches, req.waves);
  if (budget < 2 || budget % 2) throw ConfigError("chimera-wave: device budget must be even");
  if (microbatches % 2) throw ConfigError("chimera-wave: B must be even");
  ScheduleConfig cfg = make_config(Scheme::ChimeraWave, budget / 2, microbatches / 2, req.waves, 2);
  *cost = base.rescaled(budget, cfg.devices);
  return cfg;
}

bool row_before(const CompareRow& a, const CompareRow& b) {
  if (a.failed != b.failed) return b.failed;
  if (!a.failed && a.makespan != b.makespan) return a.makespan < b.makespan;
  if (a.scheme != b.scheme) return static_cast<int>(a.scheme) < static_cast<int>(b.scheme);
  return a.waves < b.waves;
}

// JSON number as the reference's nlohmann dump writes a double: shortest
// round trip, ".0" on integral values.
std::string json_num(double v) {
  char b[64];
  auto e = std::to_chars(b, b + sizeof b, v);
  std::string s(b, e.ptr);
  if (std::isfinite(v) && s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s;
}

std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      case '\t': o += "\\t"; break;
      case '\r': o += "\\r"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char u[8];
          std::snprintf(u, sizeof u, "\\u%04x", c);
          o += u;
        } else {
          o += c;
        }
    }
  }
  return o + "\"";
}

}  // namespace

std::vector<CompareRow> compare(const std::vector<CompareRequest>& requests, int budget_devices, int microbatches,
                                const CostModel& base_cost) {
  std::vector<CompareRow> rows;
  rows.reserve(requests.size());
  for (const CompareRequest& req : requests) {
    CompareRow row;
    row.scheme = req.scheme;
    row.devices = budget_devices;
    row.microbatches = microbatches;
    row.waves = req.waves;
    try {
      CostModel cost;
      const ScheduleConfig cfg = row_config(req, budget_devices, microbatches, base_cost, &cost);
      const ActionList list = generate_schedule(make_placement(cfg), cfg, cost);
      const MetricsReport m = compute_metrics(simulate(list, cost), list);
      row.makespan = m.makespan;
      row.simulated_ratio = m.bubble_ratio;
      if (req.scheme == Scheme::Hanayo && cfg.devices >= 2) {
        row.has_analytic = true;
        row.analytic_ratio = analytic_bubble_hanayo_d(cfg.devices, cfg.waves, cost.t_forward, cost.t_backward,
                                                      cost.t_comm);
      }
      for (const Rational& w : m.memory.weight_units) row.weight_units = std::max(row.weight_units, w);
      for (const Rational& a : m.memory.peak_activation_units) row.peak_activation = std::max(row.peak_activation, a);
      row.variance = m.activation_variance;
    } catch (const std::exception& e) {
      row.failed = true;
      row.error = e.what();
    }
    rows.push_back(std::move(row));
  }
  std::sort(rows.begin(), rows.end(), row_before);
  return rows;
}

std::vector<CompareRow> compare_measured(const std::vector<CompareRequest>& requests, int budget_devices,
                                         int microbatches, const std::vector<SimTrace>& traces,
                                         const std::vector<ActionList>& lists, double t_comm) {
  if (traces.size() != requests.size() || lists.size() != requests.size()) {
    throw std::invalid_argument("compare_measured: one trace and one list per request");
  }
  std::vector<CompareRow> rows;
  for (size_t i = 0; i < requests.size(); ++i) {
    CompareRow row;
    row.scheme = requests[i].scheme;
    row.devices = budget_devices;
    row.microbatches = microbatches;
    row.waves = requests[i].waves;
    try {
      const MetricsReport m = compute_metrics(traces[i], lists[i]);
      row.makespan = m.makespan;
      row.simulated_ratio = m.bubble_ratio;
      const ScheduleConfig& cfg = lists[i].config;
      if (row.scheme == Scheme::Hanayo && cfg.devices >= 2) {
        // Mean measured slice durations, scaled to stage costs (a slice is
        // 1/(2W) of a stage, ref include/wavepipe/cost_model.hpp:32-37).
        double f = 0, b = 0;
        int nf = 0, nb = 0;
        for (const auto& dev : traces[i].intervals)
          for (const TraceInterval& iv : dev) {
            if (iv.kind == ActionKind::Forward) f += iv.end - iv.start, ++nf;
            if (iv.kind == ActionKind::Backward) b += iv.end - iv.start, ++nb;
          }
        if (nf && nb) {
          row.has_analytic = true;
          row.analytic_ratio = analytic_bubble_hanayo_d(cfg.devices, cfg.waves, 2.0 * cfg.waves * f / nf,
                                                        2.0 * cfg.waves * b / nb, t_comm);
        }
      }
      for (const Rational& w : m.memory.weight_units) row.weight_units = std::max(row.weight_units, w);
      for (const Rational& a : m.memory.peak_activation_units) row.peak_activation = std::max(row.peak_activation, a);
      row.variance = m.activation_variance;
    } catch (const std::exception& e) {
      row.failed = true;
      row.error = e.what();
    }
    rows.push_back(std::move(row));
  }
  std::sort(rows.begin(), rows.end(), row_before);
  return rows;
}

std::string compare_to_csv(const std::vector<CompareRow>& rows) {
  std::ostringstream os;
  os << "scheme,devices,microbatches,waves,makespan,simulated_bubble_ratio,analytic_bubble_ratio,weight_units,"
        "peak_activation_units,activation_variance,error\n";
  for (const CompareRow& r : rows) {
    os << scheme_name(r.scheme) << ',' << r.devices << ',' << r.microbatches << ',' << r.waves << ',';
    if (r.failed) {
      std::string msg = r.error;
      std::replace(msg.begin(), msg.end(), ',', ';');
      os << ",,,,,," << msg << '\n';
      continue;
    }
    os << r.makespan << ',' << r.simulated_ratio << ',';
    if (r.has_analytic) os << r.analytic_ratio;
    os << ',' << r.weight_units.to_string() << ',' << r.peak_activation.to_string() << ','
       << r.variance.to_string() << ",\n";
  }
  return os.str();
}

std::string compare_to_json(const std::vector<CompareRow>& rows) {
  if (rows.empty()) return "[]\n";
  std::string o = "[";
  for (size_t i = 0; i < rows.size(); ++i) {
    const CompareRow& r = rows[i];
    o += i ? ",\n  {" : "\n  {";
    o += "\n    \"scheme\": " + json_str(scheme_name(r.scheme)) + ",\n    \"devices\": " +
         std::to_string(r.devices) + ",\n    \"microbatches\": " + std::to_string(r.microbatches) +
         ",\n    \"waves\": " + std::to_string(r.waves);
    if (r.failed) {
      o += ",\n    \"error\": " + json_str(r.error);
    } else {
      o += ",\n    \"makespan\": " + json_num(r.makespan) + ",\n    \"simulated_bubble_ratio\": " +
           json_num(r.simulated_ratio) + ",\n    \"analytic_bubble_ratio\": " +
           (r.has_analytic ? json_num(r.analytic_ratio) : std::string("null")) + ",\n    \"weight_units\": " +
           json_str(r.weight_units.to_string()) + ",\n    \"peak_activation_units\": " +
           json_str(r.peak_activation.to_string()) + ",\n    \"activation_variance\": " +
           json_str(r.variance.to_string());
    }
    o += "\n  }";
  }
  return o + "\n]\n";
}

}  // namespace wavepipe
