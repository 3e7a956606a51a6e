// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A small command-line driver linked against the UNMODIFIED reference
// sources under /root/reference/proj/src (compiled in place by
// oracle/Makefile; nothing is copied into this repo).  It exposes the
// reference's schedule path -- make_config (src/config.cpp:47), make_placement
// (src/placement.cpp:70), generate_schedule (src/schedule.cpp:475), simulate
// (src/simulate.cpp:57), bubble_ratio / memory_profile / analytic_bubble_*
// (src/analytics.cpp:32,48,124,159) and serialize_action_list
// (src/serialize.cpp:236) -- so tests/golden/make_golden.py can freeze its
// outputs and bench.py's reference arm can time it.
//
// Commands (all output on stdout):
//   dump  <scheme> P B W D tf tb tc   compact JSON: actions, trace, metrics
//   json  <scheme> P B W D tf tb tc   stock serialize_action_list text
//   regen <file.json>                  regenerate a stored golden, print JSON
//   eq1   P W tf tb tc                 analytic_bubble_hanayo_d
//   time  <scheme> P B W reps          best-of-reps ms of generate+simulate
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>

#include "wavepipe/gantt.hpp"
#include "wavepipe/analytics.hpp"
#include "wavepipe/placement.hpp"
#include "wavepipe/schedule.hpp"
#include "wavepipe/serialize.hpp"
#include "wavepipe/simulate.hpp"

using namespace wavepipe;

static Scheme parse_scheme(const char* s) {
  Scheme out;
  if (!scheme_from_name(s, &out)) {
    std::fprintf(stderr, "unknown scheme %s\n", s);
    std::exit(2);
  }
  return out;
}

static void print_dump(const ActionList& list, const CostModel& cost) {
  SimTrace tr = simulate(list, cost);
  std::printf("{\"actions\":[");
  for (size_t d = 0; d < list.per_device.size(); ++d) {
    std::printf(d ? ",[" : "[");
    for (size_t i = 0; i < list.per_device[d].size(); ++i) {
      const Action& a = list.per_device[d][i];
      std::printf("%s[%d,%d,%d,%d,%d,%d,%d]", i ? "," : "", static_cast<int>(a.kind),
                  a.microbatch, a.local_module_rank, a.slice_index, a.peer,
                  a.payload, a.batch_group);
    }
    std::printf("]");
  }
  std::printf("],\"makespan\":%.17g", tr.makespan);
  std::printf(",\"bubble\":%.17g", tr.makespan > 0 ? bubble_ratio(tr) : 0.0);
  MemoryProfile mp = memory_profile(tr, list);
  std::printf(",\"peaks\":[");
  for (size_t d = 0; d < mp.peak_activation_units.size(); ++d) {
    std::printf("%s[%lld,%lld]", d ? "," : "",
                static_cast<long long>(mp.peak_activation_units[d].num()),
                static_cast<long long>(mp.peak_activation_units[d].den()));
  }
  std::printf("],\"weights\":[");
  for (size_t d = 0; d < mp.weight_units.size(); ++d) {
    std::printf("%s[%lld,%lld]", d ? "," : "",
                static_cast<long long>(mp.weight_units[d].num()),
                static_cast<long long>(mp.weight_units[d].den()));
  }
  std::printf("],\"intervals\":[");
  for (size_t d = 0; d < tr.intervals.size(); ++d) {
    std::printf(d ? ",[" : "[");
    for (size_t i = 0; i < tr.intervals[d].size(); ++i) {
      const TraceInterval& iv = tr.intervals[d][i];
      std::printf("%s[%d,%d,%d,%d,%.17g,%.17g]", i ? "," : "", iv.action_index,
                  static_cast<int>(iv.kind), iv.microbatch, iv.slice_index,
                  iv.start, iv.end);
    }
    std::printf("]");
  }
  std::printf("],\"comm_events\":[");
  for (size_t i = 0; i < tr.comm_events.size(); ++i) {
    const CommEvent& e = tr.comm_events[i];
    std::printf("%s[%d,%d,%.17g,%.17g]", i ? "," : "", e.src_device, e.dst_device,
                e.post_time, e.arrival_time);
  }
  std::printf("]}\n");
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_driver dump|json|regen|eq1|time ...\n");
    return 2;
  }
  std::string cmd = argv[1];
  try {
    if ((cmd == "dump" || cmd == "json") && argc == 10) {
      ScheduleConfig cfg = make_config(parse_scheme(argv[2]), std::atoi(argv[3]),
                                       std::atoi(argv[4]), std::atoi(argv[5]),
                                       std::atoi(argv[6]));
      CostModel cost;
      cost.t_forward = std::atof(argv[7]);
      cost.t_backward = std::atof(argv[8]);
      cost.t_comm = std::atof(argv[9]);
      ActionList list = generate_schedule(make_placement(cfg), cfg, cost);
      if (cmd == "json") {
        std::fputs(serialize_action_list(list).c_str(), stdout);
      } else {
        print_dump(list, cost);
      }
      return 0;
    }
    if (cmd == "regen" && argc == 3) {
      std::ifstream in(argv[2], std::ios::binary);
      std::ostringstream os;
      os << in.rdbuf();
      ActionList stored = parse_action_list(os.str());
      ActionList fresh = generate_schedule(stored.placement, stored.config, CostModel{});
      std::fputs(serialize_action_list(fresh).c_str(), stdout);
      return 0;
    }
    if (cmd == "gantt" && argc == 4) {  // gantt <golden.json> svg|csv: the reference's own renderer
      std::ifstream in(argv[2], std::ios::binary);
      std::ostringstream os;
      os << in.rdbuf();
      ActionList stored = parse_action_list(os.str());
      std::fputs(trace_to_gantt(simulate(stored, CostModel{}), argv[3]).c_str(), stdout);
      return 0;
    }
    if (cmd == "eq1" && argc == 7) {
      std::printf("%.17g\n", analytic_bubble_hanayo_d(std::atoi(argv[2]), std::atoi(argv[3]),
                                                      std::atof(argv[4]), std::atof(argv[5]),
                                                      std::atof(argv[6])));
      return 0;
    }
    if (cmd == "compare" && argc >= 9) {  // compare P B tf tb tc csv|json scheme:waves...
      std::vector<CompareRequest> reqs;
      for (int i = 8; i < argc; ++i) {
        std::string a = argv[i];
        const size_t colon = a.find(':');
        CompareRequest r;
        r.scheme = parse_scheme(a.substr(0, colon).c_str());
        r.waves = colon == std::string::npos ? 1 : std::atoi(a.c_str() + colon + 1);
        reqs.push_back(r);
      }
      CostModel cost;
      cost.t_forward = std::atof(argv[4]);
      cost.t_backward = std::atof(argv[5]);
      cost.t_comm = std::atof(argv[6]);
      const auto rows = compare(reqs, std::atoi(argv[2]), std::atoi(argv[3]), cost);
      std::fputs((std::string(argv[7]) == "csv" ? compare_to_csv(rows) : compare_to_json(rows)).c_str(), stdout);
      return 0;
    }
    if (cmd == "time" && argc == 7) {
      ScheduleConfig cfg = make_config(parse_scheme(argv[2]), std::atoi(argv[3]),
                                       std::atoi(argv[4]), std::atoi(argv[5]), 1);
      int reps = std::atoi(argv[6]);
      double best = 1e30;
      double sink = 0;
      for (int r = 0; r < reps; ++r) {
        auto t0 = std::chrono::steady_clock::now();
        ActionList list = generate_schedule(make_placement(cfg), cfg, CostModel{});
        SimTrace tr = simulate(list, CostModel{});
        sink += tr.makespan;
        auto t1 = std::chrono::steady_clock::now();
        double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        if (ms < best) best = ms;
      }
      std::printf("{\"best_ms\":%.6f,\"reps\":%d,\"makespan\":%.17g}\n", best, reps,
                  sink / reps);
      return 0;
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "bad arguments\n");
  return 2;
}
