// C ABI over the schedule path (include/wavepipe.h).  Every entry point
// catches, maps the exception type to the reference CLI's exit-code taxonomy
// (tools/main.cpp:37-40, :297-312) and stores the message for wp_last_error.
#include <algorithm>
#include <cstring>
#include <string>

#include "capi_internal.hpp"
#include "wavepipe.h"

namespace wpc {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int map_exception() {
  try {
    throw;
  } catch (const wavepipe::ConfigError& e) {
    return fail(WP_ERR_CONFIG, e.what());
  } catch (const wavepipe::ParseError& e) {
    return fail(WP_ERR_CONFIG, e.what());
  } catch (const wavepipe::ScheduleError& e) {
    return fail(WP_ERR_SEMANTIC, e.what());
  } catch (const wavepipe::SimulationError& e) {
    return fail(WP_ERR_SEMANTIC, e.what());
  } catch (const CudaError& e) {
    return fail(WP_ERR_CUDA, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(WP_ERR_CONFIG, e.what());
  } catch (const std::exception& e) {
    return fail(WP_ERR_SEMANTIC, e.what());
  } catch (...) {
    return fail(WP_ERR_SEMANTIC, "unknown error");
  }
}

void refresh(wp_list* l) {
  l->flat.assign(l->list.per_device.size(), {});
  for (size_t d = 0; d < l->list.per_device.size(); ++d) {
    for (const auto& a : l->list.per_device[d]) {
      l->flat[d].push_back(wp_action{static_cast<int>(a.kind), a.microbatch, a.local_module_rank,
                                     a.slice_index, a.peer, a.payload, a.batch_group});
    }
  }
}

void refresh(wp_trace* t) {
  t->flat.assign(t->trace.intervals.size(), {});
  for (size_t d = 0; d < t->trace.intervals.size(); ++d) {
    for (const auto& iv : t->trace.intervals[d]) {
      t->flat[d].push_back(wp_interval{iv.action_index, static_cast<int>(iv.kind), iv.microbatch,
                                       iv.slice_index, static_cast<int>(iv.direction), iv.start, iv.end});
    }
  }
  t->events.clear();
  for (const auto& e : t->trace.comm_events) {
    t->events.push_back(wp_comm_event{e.src_device, e.dst_device, e.post_time, e.arrival_time});
  }
}

wavepipe::ScheduleConfig to_cfg(const wp_config& c) {
  if (c.scheme < 0 || c.scheme > 4) throw wavepipe::ConfigError("unknown scheme value");
  return wavepipe::make_config(static_cast<wavepipe::Scheme>(c.scheme), c.devices, c.microbatches,
                               c.waves, c.replicas);
}

wavepipe::CostModel to_cost(const wp_cost* c) {
  wavepipe::CostModel m;
  if (c) {
    m.t_forward = c->t_forward;
    m.t_backward = c->t_backward;
    m.t_comm = c->t_comm;
  }
  return m;
}

}  // namespace wpc

using namespace wpc;

extern "C" {

const char* wp_last_error(void) { return g_last_error.c_str(); }
const char* wp_version(void) { return "wavepipe-b200 0.1 (sm_100a)"; }

int wp_make_config(int scheme, int P, int B, int W, int D, wp_config* out) {
  try {
    if (!out) return fail(WP_ERR_CONFIG, "null output");
    if (scheme < 0 || scheme > 4) return fail(WP_ERR_CONFIG, "unknown scheme value");
    const auto c = wavepipe::make_config(static_cast<wavepipe::Scheme>(scheme), P, B, W, D);
    *out = wp_config{static_cast<int>(c.scheme), c.devices, c.microbatches, c.waves, c.replicas, c.stages};
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_generate_schedule(const wp_config* cfg, const wp_cost* cost, wp_list** out) {
  try {
    if (!cfg || !out) return fail(WP_ERR_CONFIG, "null argument");
    const auto c = to_cfg(*cfg);
    auto* l = new wp_list;
    try {
      l->list = wavepipe::generate_schedule(wavepipe::make_placement(c), c, to_cost(cost));
    } catch (...) {
      delete l;
      throw;
    }
    refresh(l);
    *out = l;
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_list_from_actions(const wp_config* cfg, const int* counts, const wp_action* actions, wp_list** out) {
  try {
    if (!cfg || !counts || !out) return fail(WP_ERR_CONFIG, "null argument");
    const auto c = to_cfg(*cfg);
    auto* l = new wp_list;
    l->list.config = c;
    l->list.placement = wavepipe::make_placement(c);
    l->list.per_device.resize(c.devices);
    size_t k = 0;
    for (int d = 0; d < c.devices; ++d) {
      for (int i = 0; i < counts[d]; ++i, ++k) {
        const wp_action& w = actions[k];
        if (w.kind < 0 || w.kind > 5) {
          delete l;
          return fail(WP_ERR_CONFIG, "unknown action kind value");
        }
        wavepipe::Action a;
        a.kind = static_cast<wavepipe::ActionKind>(w.kind);
        a.microbatch = w.microbatch;
        a.local_module_rank = w.local_module_rank;
        a.slice_index = w.slice_index;
        a.peer = w.peer;
        a.payload = w.payload;
        a.batch_group = w.batch_group;
        l->list.per_device[d].push_back(a);
      }
    }
    refresh(l);
    *out = l;
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_insert_comm(const wp_list* in, wp_list** out) {
  try {
    if (!in || !out) return fail(WP_ERR_CONFIG, "null argument");
    auto* l = new wp_list;
    try {
      l->list = wavepipe::insert_comm(in->list);
    } catch (...) {
      delete l;
      throw;
    }
    refresh(l);
    *out = l;
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_list_config(const wp_list* l, wp_config* out) {
  if (!l || !out) return fail(WP_ERR_CONFIG, "null argument");
  const auto& c = l->list.config;
  *out = wp_config{static_cast<int>(c.scheme), c.devices, c.microbatches, c.waves, c.replicas, c.stages};
  return WP_OK;
}

int wp_list_device(const wp_list* l, int d, const wp_action** actions, int* count) {
  if (!l || !actions || !count) return fail(WP_ERR_CONFIG, "null argument");
  if (d < 0 || d >= static_cast<int>(l->flat.size())) return fail(WP_ERR_CONFIG, "device out of range");
  *actions = l->flat[d].data();
  *count = static_cast<int>(l->flat[d].size());
  return WP_OK;
}

int wp_list_placement(const wp_list* l, int d, int* idx, int cap, int* count) {
  if (!l || !count) return fail(WP_ERR_CONFIG, "null argument");
  const auto& as = l->list.placement.assignment;
  if (d < 0 || d >= static_cast<int>(as.size())) return fail(WP_ERR_CONFIG, "device out of range");
  *count = static_cast<int>(as[d].size());
  for (int i = 0; i < *count && i < cap && idx; ++i) idx[i] = as[d][i].index;
  return WP_OK;
}

void wp_list_free(wp_list* l) { delete l; }

int wp_serialize(const wp_list* l, char** json) {
  try {
    if (!l || !json) return fail(WP_ERR_CONFIG, "null argument");
    const std::string s = wavepipe::serialize_action_list(l->list);
    char* buf = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(buf, s.c_str(), s.size() + 1);
    *json = buf;
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

namespace {
char* dup_c(const std::string& s) {
  char* buf = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return buf;
}
std::vector<wavepipe::CompareRequest> requests_of(const int* schemes, const int* waves, int n) {
  std::vector<wavepipe::CompareRequest> r(n);
  for (int i = 0; i < n; ++i) {
    if (schemes[i] < 0 || schemes[i] > static_cast<int>(wavepipe::Scheme::Hanayo)) {
      throw wavepipe::ConfigError("compare: unknown scheme " + std::to_string(schemes[i]));
    }
    r[i].scheme = static_cast<wavepipe::Scheme>(schemes[i]);
    r[i].waves = waves[i];
  }
  return r;
}
}  // namespace

int wp_compare(const int* schemes, const int* waves, int n, int budget_devices, int microbatches,
               const wp_cost* base_cost, int format, char** out) {
  try {
    if ((n > 0 && (!schemes || !waves)) || !base_cost || !out) return fail(WP_ERR_CONFIG, "null argument");
    wavepipe::CostModel c;
    c.t_forward = base_cost->t_forward, c.t_backward = base_cost->t_backward, c.t_comm = base_cost->t_comm;
    const auto rows = wavepipe::compare(requests_of(schemes, waves, n), budget_devices, microbatches, c);
    *out = dup_c(format == 1 ? wavepipe::compare_to_json(rows) : wavepipe::compare_to_csv(rows));
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_compare_measured(const int* schemes, const int* waves, int n, int budget_devices, int microbatches,
                        const wp_trace* const* traces, const wp_list* const* lists, double t_comm, int format,
                        char** out) {
  try {
    if ((n > 0 && (!schemes || !waves || !traces || !lists)) || !out) return fail(WP_ERR_CONFIG, "null argument");
    std::vector<wavepipe::SimTrace> tr;
    std::vector<wavepipe::ActionList> ls;
    for (int i = 0; i < n; ++i) {
      if (!traces[i] || !lists[i]) return fail(WP_ERR_CONFIG, "null trace or list");
      tr.push_back(traces[i]->trace);
      ls.push_back(lists[i]->list);
    }
    const auto rows = wavepipe::compare_measured(requests_of(schemes, waves, n), budget_devices, microbatches, tr, ls,
                                                 t_comm);
    *out = dup_c(format == 1 ? wavepipe::compare_to_json(rows) : wavepipe::compare_to_csv(rows));
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_trace_to_gantt(const wp_trace* t, const char* format, char** out) {
  try {
    if (!t || !format || !out) return fail(WP_ERR_CONFIG, "null argument");
    const std::string s = wavepipe::trace_to_gantt(t->trace, format);
    char* buf = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(buf, s.c_str(), s.size() + 1);
    *out = buf;
    return WP_OK;
  } catch (const std::invalid_argument& e) {
    return fail(WP_ERR_CONFIG, e.what());
  } catch (...) {
    return map_exception();
  }
}

int wp_parse(const char* json, wp_list** out) {
  try {
    if (!json || !out) return fail(WP_ERR_CONFIG, "null argument");
    auto* l = new wp_list;
    try {
      l->list = wavepipe::parse_action_list(json);
    } catch (...) {
      delete l;
      throw;
    }
    refresh(l);
    *out = l;
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

void wp_string_free(char* s) { std::free(s); }

int wp_validate(const wp_list* l, int* ok, char* report, int capacity) {
  try {
    if (!l || !ok) return fail(WP_ERR_CONFIG, "null argument");
    const auto r = wavepipe::validate_all(l->list);
    *ok = r.ok() ? 1 : 0;
    if (report && capacity > 0) {
      const std::string t = wavepipe::render_diagnostics_text(r);
      const size_t n = std::min(t.size(), size_t(capacity - 1));
      std::memcpy(report, t.data(), n);
      report[n] = 0;
    }
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_simulate(const wp_list* l, const wp_cost* cost, wp_trace** out) {
  try {
    if (!l || !out) return fail(WP_ERR_CONFIG, "null argument");
    auto* t = new wp_trace;
    try {
      t->trace = wavepipe::simulate(l->list, to_cost(cost));
    } catch (...) {
      delete t;
      throw;
    }
    refresh(t);
    *out = t;
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_trace_makespan(const wp_trace* t, double* m) {
  if (!t || !m) return fail(WP_ERR_CONFIG, "null argument");
  *m = t->trace.makespan;
  return WP_OK;
}

int wp_trace_devices(const wp_trace* t, int* n) {
  if (!t || !n) return fail(WP_ERR_CONFIG, "null argument");
  *n = static_cast<int>(t->trace.intervals.size());
  return WP_OK;
}

int wp_trace_intervals(const wp_trace* t, int d, const wp_interval** iv, int* count) {
  if (!t || !iv || !count) return fail(WP_ERR_CONFIG, "null argument");
  if (d < 0 || d >= static_cast<int>(t->flat.size())) return fail(WP_ERR_CONFIG, "device out of range");
  *iv = t->flat[d].data();
  *count = static_cast<int>(t->flat[d].size());
  return WP_OK;
}

int wp_trace_comm_events(const wp_trace* t, const wp_comm_event** ev, int* count) {
  if (!t || !ev || !count) return fail(WP_ERR_CONFIG, "null argument");
  *ev = t->events.data();
  *count = static_cast<int>(t->events.size());
  return WP_OK;
}

void wp_trace_free(wp_trace* t) { delete t; }

int wp_trace_build(int devices, const int* counts, const wp_interval* iv, int n_events, const wp_comm_event* ev,
                   wp_trace** out) {
  try {
    if (devices < 0 || n_events < 0 || !out || (devices > 0 && !counts) || (n_events > 0 && !ev)) {
      return fail(WP_ERR_CONFIG, "null or negative argument");
    }
    auto* t = new wp_trace;
    t->trace.intervals.resize(devices);
    int64_t k = 0;
    for (int d = 0; d < devices; ++d) {
      if (counts[d] < 0) {
        delete t;
        return fail(WP_ERR_CONFIG, "negative interval count");
      }
      for (int i = 0; i < counts[d]; ++i, ++k) {
        const wp_interval& x = iv[k];
        wavepipe::TraceInterval y;
        y.action_index = x.action_index;
        y.kind = static_cast<wavepipe::ActionKind>(x.kind);
        y.microbatch = x.microbatch;
        y.slice_index = x.slice_index;
        y.direction = static_cast<wavepipe::Direction>(x.direction);
        y.start = x.start;
        y.end = x.end;
        t->trace.makespan = std::max(t->trace.makespan, y.end);
        t->trace.intervals[d].push_back(y);
      }
    }
    for (int i = 0; i < n_events; ++i) {
      t->trace.comm_events.push_back(
          wavepipe::CommEvent{ev[i].src_device, ev[i].dst_device, ev[i].post_time, ev[i].arrival_time});
      t->trace.makespan = std::max(t->trace.makespan, ev[i].arrival_time);
    }
    refresh(t);
    *out = t;
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_bubble_ratio(const wp_trace* t, double* out) {
  try {
    if (!t || !out) return fail(WP_ERR_CONFIG, "null argument");
    *out = wavepipe::bubble_ratio(t->trace);
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_memory_profile(const wp_trace* t, const wp_list* l, int64_t* w, int64_t* peak) {
  try {
    if (!t || !l) return fail(WP_ERR_CONFIG, "null argument");
    const auto mp = wavepipe::memory_profile(t->trace, l->list);
    for (size_t d = 0; d < mp.weight_units.size(); ++d) {
      if (w) {
        w[2 * d] = mp.weight_units[d].num();
        w[2 * d + 1] = mp.weight_units[d].den();
      }
      if (peak) {
        peak[2 * d] = mp.peak_activation_units[d].num();
        peak[2 * d + 1] = mp.peak_activation_units[d].den();
      }
    }
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_analytic_bubble(int P, int W, double tf, double tb, double tc, double* out) {
  try {
    if (!out) return fail(WP_ERR_CONFIG, "null argument");
    *out = wavepipe::analytic_bubble_hanayo_d(P, W, tf, tb, tc);
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_analytic_bubble_exact(int P, int W, const int64_t tf[2], const int64_t tb[2], const int64_t tc[2],
                             int64_t out[2]) {
  try {
    if (!tf || !tb || !tc || !out) return fail(WP_ERR_CONFIG, "null argument");
    const auto r = wavepipe::analytic_bubble_hanayo(P, W, wavepipe::Rational(tf[0], tf[1]),
                                                    wavepipe::Rational(tb[0], tb[1]),
                                                    wavepipe::Rational(tc[0], tc[1]));
    out[0] = r.num();
    out[1] = r.den();
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_analytic_bubble_simplified(int P, int W, int64_t out[2]) {
  try {
    if (!out) return fail(WP_ERR_CONFIG, "null argument");
    const auto r = wavepipe::analytic_bubble_simplified(P, W);
    out[0] = r.num();
    out[1] = r.den();
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

}  // extern "C"
