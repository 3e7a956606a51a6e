// A reference-API caller (include names of proj/include/wavepipe) driving the
// GPU train step: generate the Hanayo list exactly as the reference would,
// run wavepipe::train_step, and feed the measured trace to the reference's
// analytics and Gantt renderer unchanged.
#include <cmath>
#include <cstdio>
#include <vector>

#include "wavepipe/analytics.hpp"
#include "wavepipe/config.hpp"
#include "wavepipe/gantt.hpp"
#include "wavepipe/placement.hpp"
#include "wavepipe/runtime.hpp"
#include "wavepipe/schedule.hpp"

int main() {
  using namespace wavepipe;
  const ScheduleConfig cfg = make_config(Scheme::Hanayo, 2, 4, 2);
  const ActionList list = generate_schedule(make_placement(cfg), cfg, CostModel{});
  ModelSpec m;
  m.layers = 2;
  m.bf16 = true;
  m.adamw = true;
  Runtime rt(m, list, Transport::Local, {0, 0});
  const int n = cfg.microbatches * m.micro_batch_size * m.seq;
  std::vector<int32_t> tok(n), lab(n);
  for (int i = 0; i < n; ++i) {
    tok[i] = (i * 7919) % m.vocab;
    lab[i] = (i * 104729 + 1) % m.vocab;
  }
  float first = 0.f;
  for (int step = 0; step < 3; ++step) {
    const SimTrace tr = train_step(list, rt, Batch{tok.data(), lab.data(), false});
    if (step == 0) first = rt.last_loss();
    int intervals = 0;
    for (const auto& d : tr.intervals) intervals += static_cast<int>(d.size());
    const std::string csv = trace_to_gantt(tr, "csv");
    std::printf("step %d loss %.5f makespan %.6f s bubble %.4f intervals %d gantt_bytes %zu\n", step, rt.last_loss(),
                tr.makespan, bubble_ratio(tr), intervals, csv.size());
    if (!std::isfinite(rt.last_loss()) || intervals != 2 * cfg.microbatches * cfg.stages) return 1;
  }
  return rt.last_loss() < first ? 0 : 2;  // AdamW on a fixed batch lowers the loss
}
