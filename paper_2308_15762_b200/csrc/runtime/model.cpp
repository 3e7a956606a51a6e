#include "runtime/model.hpp"

#include <cmath>
#include <utility>
#include <stdexcept>

#include "wavepipe/core.hpp"

namespace wprt {

ModelSpec ModelSpec::from_desc(const wp_model_desc& d) {
  ModelSpec m{};
  m.layers = d.layers;
  m.hidden = d.hidden;
  m.heads = d.heads;
  m.ffn = d.ffn;
  m.seq = d.seq;
  m.vocab = d.vocab;
  m.mbs = d.micro_batch_size;
  m.causal = d.causal != 0;
  m.tie = d.tie_embeddings != 0;
  m.dtype = d.dtype;
  m.optimizer = d.optimizer;
  m.lr = d.lr;
  m.beta1 = d.beta1;
  m.beta2 = d.beta2;
  m.eps = d.eps;
  m.weight_decay = d.weight_decay;
  m.seed = d.seed;
  auto need = [](bool ok, const char* msg) {
    if (!ok) throw wavepipe::ConfigError(std::string("model: ") + msg);
  };
  need(m.layers >= 1 && m.hidden > 0 && m.heads > 0 && m.ffn > 0 && m.seq > 0 && m.vocab > 0 && m.mbs > 0,
       "all sizes must be positive");
  need(m.hidden % m.heads == 0, "hidden must divide by heads");
  need(m.hidden % 256 == 0 && m.hidden <= 4096, "hidden must be a multiple of 256, at most 4096");
  need(m.ffn % 8 == 0 && m.vocab % 8 == 0, "ffn and vocab must be multiples of 8");
  need(m.seq <= 1024 && m.seq % 8 == 0, "seq must be a multiple of 8, at most 1024");
  need(m.head_dim() % 8 == 0, "head_dim must be a multiple of 8");
  need(m.dtype == 0 || m.dtype == 1, "dtype must be 0 (fp32) or 1 (bf16)");
  need(m.optimizer == 0 || m.optimizer == 1, "optimizer must be 0 (SGD) or 1 (AdamW)");
  return m;
}

std::vector<Unit> build_units(const ModelSpec& m) {
  const double h = m.hidden, f = m.ffn, s = m.seq, V = m.vocab;
  const double attn_core = (m.causal ? 2.0 : 4.0) * s * h;  // QK^T + PV per token (causal halves)
  std::vector<Unit> u;
  u.push_back({UnitKind::Embed, -1, h});
  for (int l = 0; l < m.layers; ++l) {
    u.push_back({UnitKind::Attn, l, 8.0 * h * h + attn_core});
    u.push_back({UnitKind::Mlp, l, 4.0 * h * f});
  }
  u.push_back({UnitKind::Head, -1, 2.0 * h * V});
  return u;
}

std::vector<int> partition_units(const std::vector<Unit>& units, int S) {
  const int N = static_cast<int>(units.size());
  std::vector<double> prefix(N + 1, 0.0);
  for (int i = 0; i < N; ++i) prefix[i + 1] = prefix[i] + units[i].cost;
  const double total = prefix[N];
  std::vector<int> b(S + 1, 0);
  b[0] = 0;
  b[S] = N;
  for (int k = 1; k < S; ++k) {
    const double target = total * k / S;
    // Cuts lie in [1, N-1]: slice 0 keeps the embedding, slice S-1 the head.
    int lo = std::max(b[k - 1], 1), best = lo;
    double best_d = std::fabs(prefix[lo] - target);
    for (int i = lo + 1; i <= N - 1; ++i) {
      const double d = std::fabs(prefix[i] - target);
      if (d < best_d) {
        best = i;
        best_d = d;
      }
    }
    b[k] = std::min(best, N - 1);
  }
  return b;
}

std::vector<int> partition_units(const std::vector<Unit>& units, const std::vector<int>& slice_device, int P) {
  const int S = static_cast<int>(slice_device.size());
  const int N = static_cast<int>(units.size());
  std::vector<double> prefix(N + 1, 0.0);
  for (int i = 0; i < N; ++i) prefix[i + 1] = prefix[i] + units[i].cost;
  const double total = prefix[N];
  // Per-slice targets: every device gets total / P; the pinned units (the
  // embedding in slice 0, the LM head in slice S-1) count toward their
  // device, whose other slices share what is left of its budget.
  std::vector<double> fixed(S, 0.0), dev_fixed(P, 0.0);
  std::vector<int> dev_slices(P, 0);
  fixed[0] += units.front().cost;
  fixed[S - 1] += units.back().cost;
  for (int k = 0; k < S; ++k) {
    dev_fixed[slice_device[k]] += fixed[k];
    ++dev_slices[slice_device[k]];
  }
  std::vector<double> target(S);
  double tsum = 0.0;
  for (int k = 0; k < S; ++k) {
    const int d = slice_device[k];
    target[k] = fixed[k] + std::max(0.0, total / P - dev_fixed[d]) / dev_slices[d];
    tsum += target[k];
  }
  std::vector<int> b(S + 1, 0);
  b[S] = N;
  double cum = 0.0;
  for (int k = 1; k < S; ++k) {
    cum += target[k - 1] * total / tsum;
    int lo = std::max(b[k - 1], 1), best = lo;
    double best_d = std::fabs(prefix[lo] - cum);
    for (int i = lo + 1; i <= N - 1; ++i) {
      const double dd = std::fabs(prefix[i] - cum);
      if (dd < best_d) best = i, best_d = dd;
    }
    b[k] = std::min(best, N - 1);
  }
  // Coordinate descent on the cuts: each cut moves to the position that
  // minimises (max device load, sum of squared device loads) until no cut
  // moves.  Pipeline throughput is bounded by the busiest device.
  auto score = [&](const std::vector<int>& bb) {
    std::vector<double> load(P, 0.0);
    for (int k = 0; k < S; ++k) load[slice_device[k]] += prefix[bb[k + 1]] - prefix[bb[k]];
    double mx = 0.0, sq = 0.0;
    for (double l : load) mx = std::max(mx, l), sq += l * l;
    return std::make_pair(mx, sq);
  };
  auto cur = score(b);
  for (bool moved = true; moved;) {
    moved = false;
    for (int k = 1; k < S; ++k) {
      const int lo = std::max(b[k - 1], 1), hi = std::min(b[k + 1], N - 1);
      int best = b[k];
      auto best_s = cur;
      for (int pos = lo; pos <= hi; ++pos) {
        b[k] = pos;
        const auto sc = score(b);
        if (sc < best_s) best_s = sc, best = pos;
      }
      b[k] = best;
      if (best_s < cur) {
        cur = best_s;
        moved = true;
      }
    }
  }
  return b;
}

std::vector<ParamDesc> unit_params(const ModelSpec& m, int ui, const Unit& u) {
  const int64_t h = m.hidden, f = m.ffn, V = m.vocab, s = m.seq;
  const float std_w = 0.02f;
  const float std_out = 0.02f / std::sqrt(2.0f * m.layers);  // GPT-2 residual projection scaling
  std::vector<ParamDesc> p;
  auto add = [&](std::string name, std::vector<int64_t> shape, float sd, float val) {
    ParamDesc d;
    d.name = std::move(name);
    d.shape = shape;
    d.numel = 1;
    for (auto x : shape) d.numel *= x;
    d.unit = ui;
    d.init_std = sd;
    d.init_value = val;
    p.push_back(d);
  };
  const std::string L = "h." + std::to_string(u.layer) + ".";
  switch (u.kind) {
    case UnitKind::Embed:
      add("wte", {V, h}, std_w, 0);
      add("wpe", {s, h}, std_w, 0);
      break;
    case UnitKind::Attn:
      add(L + "ln1.w", {h}, 0, 1);
      add(L + "ln1.b", {h}, 0, 0);
      add(L + "attn.qkv.w", {3 * h, h}, std_w, 0);
      add(L + "attn.qkv.b", {3 * h}, 0, 0);
      add(L + "attn.proj.w", {h, h}, std_out, 0);
      add(L + "attn.proj.b", {h}, 0, 0);
      break;
    case UnitKind::Mlp:
      add(L + "ln2.w", {h}, 0, 1);
      add(L + "ln2.b", {h}, 0, 0);
      add(L + "mlp.fc1.w", {f, h}, std_w, 0);
      add(L + "mlp.fc1.b", {f}, 0, 0);
      add(L + "mlp.fc2.w", {h, f}, std_out, 0);
      add(L + "mlp.fc2.b", {h}, 0, 0);
      break;
    case UnitKind::Head:
      add("lnf.w", {h}, 0, 1);
      add("lnf.b", {h}, 0, 0);
      if (!m.tie) add("lm_head.w", {V, h}, std_w, 0);
      break;
  }
  return p;
}

}  // namespace wprt
