// Structural pre-flight checks of an action list, run before the runtime
// executes it (the reference CLI refuses to simulate an invalid list,
// tools/main.cpp:159-165; the GPU runtime refuses to launch one).
//
// Check semantics follow src/validate.cpp:
//   completeness   :108-166  one F and one B per (microbatch, slice), on the owner
//   dependencies   :168-389  message matching (BE carries outgoing, receives the
//                            counterpart's outgoing), dataflow realisation, and an
//                            acyclic happens-before graph with BE pairs contracted
//   deadlock_free  :391-497  adjacency-fusion certification + buffered-send replay
//   flush          :499-527  exactly one OptimizerStep, last
// Diagnostics carry the same check names and location conventions; message
// wording is this library's own.
#include <algorithm>
#include <map>
#include <set>
#include <sstream>
#include <tuple>

#include "wavepipe/core.hpp"

namespace wavepipe {

namespace {

struct Key {
  int payload, mb, low;
  bool operator<(const Key& o) const { return std::tie(payload, mb, low) < std::tie(o.payload, o.mb, o.low); }
};
struct Loc {
  int dev = -1, pos = -1;
  bool operator==(const Loc& o) const { return dev == o.dev && pos == o.pos; }
};

Key outgoing_key(const Action& a) {
  const bool act = a.payload == static_cast<int>(Payload::Activation);
  const bool out = a.kind == ActionKind::Send || a.kind == ActionKind::BatchedExchange;
  return Key{a.payload, a.microbatch,
             act ? (out ? a.slice_index : a.slice_index - 1) : (out ? a.slice_index - 1 : a.slice_index)};
}

std::string describe_key(const Key& k) {
  return std::string(k.payload == 0 ? "activation" : "gradient") + " of microbatch " +
         std::to_string(k.mb) + " across boundary " + std::to_string(k.low) + "/" +
         std::to_string(k.low + 1);
}

void note(ValidationReport* r, const char* check, int dev, int pos, std::string msg) {
  r->diagnostics.push_back(Diagnostic{check, "error", dev, pos, std::move(msg)});
}

std::map<int, std::vector<Loc>> exchange_groups(const ActionList& l) {
  std::map<int, std::vector<Loc>> g;
  for (int d = 0; d < static_cast<int>(l.per_device.size()); ++d)
    for (int i = 0; i < static_cast<int>(l.per_device[d].size()); ++i)
      if (l.per_device[d][i].kind == ActionKind::BatchedExchange) g[l.per_device[d][i].batch_group].push_back({d, i});
  return g;
}

Loc other_end(const std::vector<Loc>& ends, Loc me) { return ends[0] == me ? ends[1] : ends[0]; }

SliceOwner owner_of(const ActionList& l, int mb, int s) {
  return slice_owner(l.config, l.placement, s, microbatch_direction(l.config, mb));
}

bool in_range(const ScheduleConfig& c, const Action& a) {
  return a.microbatch >= 0 && a.microbatch < c.microbatches && a.slice_index >= 0 && a.slice_index < c.stages;
}

}  // namespace

ValidationReport check_completeness(const ActionList& l) {
  ValidationReport r;
  const ScheduleConfig& c = l.config;
  std::vector<int> nf(size_t(c.microbatches) * c.stages, 0), nb(nf.size(), 0);
  for (int d = 0; d < static_cast<int>(l.per_device.size()); ++d) {
    for (int i = 0; i < static_cast<int>(l.per_device[d].size()); ++i) {
      const Action& a = l.per_device[d][i];
      if (!a.is_compute()) continue;
      if (!in_range(c, a)) {
        note(&r, "completeness", d, i, "compute action out of range: " + describe_action(a));
        continue;
      }
      const char* phase = a.kind == ActionKind::Forward ? "forward" : "backward";
      const std::string what = std::string("(microbatch ") + std::to_string(a.microbatch) + ", slice " +
                               std::to_string(a.slice_index) + ")";
      const SliceOwner o = owner_of(l, a.microbatch, a.slice_index);
      if (o.device != d) {
        note(&r, "completeness", d, i,
             std::string("misplaced ") + phase + " " + what + ": slice is owned by device " + std::to_string(o.device));
        continue;
      }
      int& n = (a.kind == ActionKind::Forward ? nf : nb)[size_t(a.microbatch) * c.stages + a.slice_index];
      if (++n > 1) note(&r, "completeness", d, i, std::string("duplicate ") + phase + " " + what);
    }
  }
  for (int b = 0; b < c.microbatches; ++b) {
    for (int s = 0; s < c.stages; ++s) {
      const int dev = owner_of(l, b, s).device;
      const std::string what = "(microbatch " + std::to_string(b) + ", slice " + std::to_string(s) + ")";
      if (!nf[size_t(b) * c.stages + s]) note(&r, "completeness", dev, -1, "missing forward " + what);
      if (!nb[size_t(b) * c.stages + s]) note(&r, "completeness", dev, -1, "missing backward " + what);
    }
  }
  return r;
}

ValidationReport check_dependencies(const ActionList& l) {
  ValidationReport r;
  const ScheduleConfig& c = l.config;
  const int P = static_cast<int>(l.per_device.size());
  std::vector<int> base(P + 1, 0);
  for (int d = 0; d < P; ++d) base[d + 1] = base[d] + static_cast<int>(l.per_device[d].size());
  const int N = base[P];
  auto id = [&](Loc x) { return base[x.dev] + x.pos; };
  std::vector<int> rep(N);
  for (int i = 0; i < N; ++i) rep[i] = i;

  const auto groups = exchange_groups(l);
  for (const auto& [g, ends] : groups) {
    if (ends.size() != 2) {
      note(&r, "dependencies", ends[0].dev, ends[0].pos,
           "batch_group " + std::to_string(g) + " has " + std::to_string(ends.size()) +
               " participants, expected 2");
      continue;
    }
    const Action& x = l.per_device[ends[0].dev][ends[0].pos];
    const Action& y = l.per_device[ends[1].dev][ends[1].pos];
    if (x.peer != ends[1].dev || y.peer != ends[0].dev) {
      note(&r, "dependencies", ends[0].dev, ends[0].pos,
           "batch_group " + std::to_string(g) + " participants are not mutual peers");
      continue;
    }
    rep[std::max(id(ends[0]), id(ends[1]))] = std::min(id(ends[0]), id(ends[1]));
  }

  std::map<Key, std::vector<Loc>> tx, rx;
  for (int d = 0; d < P; ++d) {
    for (int i = 0; i < static_cast<int>(l.per_device[d].size()); ++i) {
      const Action& a = l.per_device[d][i];
      if (a.kind == ActionKind::Send) tx[outgoing_key(a)].push_back({d, i});
      else if (a.kind == ActionKind::Receive) rx[outgoing_key(a)].push_back({d, i});
      else if (a.kind == ActionKind::BatchedExchange) {
        tx[outgoing_key(a)].push_back({d, i});
        auto it = groups.find(a.batch_group);
        if (it != groups.end() && it->second.size() == 2) {
          const Loc o = other_end(it->second, Loc{d, i});
          rx[outgoing_key(l.per_device[o.dev][o.pos])].push_back({d, i});
        }
      }
    }
  }
  for (const auto& [k, at] : tx) {
    for (size_t j = 1; j < at.size(); ++j) note(&r, "dependencies", at[j].dev, at[j].pos, "duplicate send of " + describe_key(k));
    if (!rx.count(k)) note(&r, "dependencies", at[0].dev, at[0].pos, "unmatched send of " + describe_key(k));
  }
  for (const auto& [k, at] : rx) {
    for (size_t j = 1; j < at.size(); ++j) note(&r, "dependencies", at[j].dev, at[j].pos, "duplicate receive of " + describe_key(k));
    if (!tx.count(k)) note(&r, "dependencies", at[0].dev, at[0].pos, "unmatched receive of " + describe_key(k));
  }

  std::map<std::tuple<int, int, int>, Loc> compute;  // (bwd, mb, slice) -> first location
  for (int d = 0; d < P; ++d)
    for (int i = 0; i < static_cast<int>(l.per_device[d].size()); ++i) {
      const Action& a = l.per_device[d][i];
      if (a.is_compute() && in_range(c, a))
        compute.emplace(std::make_tuple(int(a.kind == ActionKind::Backward), a.microbatch, a.slice_index), Loc{d, i});
    }

  std::vector<std::vector<int>> out(N);
  std::vector<int> indeg(N, 0);
  auto edge = [&](int u, int v) {
    u = rep[u];
    v = rep[v];
    if (u == v) return;
    out[u].push_back(v);
    ++indeg[v];
  };
  for (int d = 0; d < P; ++d)
    for (int i = 0; i + 1 < static_cast<int>(l.per_device[d].size()); ++i) edge(base[d] + i, base[d] + i + 1);
  for (const auto& [k, at] : tx) {
    auto it = rx.find(k);
    if (it != rx.end()) edge(id(at[0]), id(it->second[0]));
  }

  auto dataflow = [&](const char* what, std::tuple<int, int, int> from, std::tuple<int, int, int> to, Key k) {
    auto pf = compute.find(from), pt = compute.find(to);
    if (pf == compute.end() || pt == compute.end()) return;
    const Loc p = pf->second, q = pt->second;
    edge(id(p), id(q));
    if (p.dev == q.dev) {
      if (p.pos >= q.pos) {
        note(&r, "dependencies", p.dev, p.pos,
             std::string(what) + " dependency of microbatch " + std::to_string(std::get<1>(from)) +
                 " not realized: producer at position " + std::to_string(p.pos) +
                 " does not precede consumer at position " + std::to_string(q.pos));
      }
      return;
    }
    auto s = tx.find(k), v = rx.find(k);
    if (s == tx.end() || v == rx.end()) {
      note(&r, "dependencies", p.dev, p.pos,
           std::string(what) + " dependency not realized: no matched send/receive pair carries the " + describe_key(k));
      return;
    }
    const Loc sl = s->second[0], rl = v->second[0];
    if (sl.dev != p.dev || sl.pos < p.pos)
      note(&r, "dependencies", sl.dev, sl.pos, "send of " + describe_key(k) + " does not follow its producer");
    if (rl.dev != q.dev || rl.pos > q.pos)
      note(&r, "dependencies", rl.dev, rl.pos, "receive of " + describe_key(k) + " does not precede its consumer");
  };
  for (int b = 0; b < c.microbatches; ++b) {
    for (int s = 0; s + 1 < c.stages; ++s) {
      dataflow("forward", {0, b, s}, {0, b, s + 1}, Key{0, b, s});
      dataflow("backward", {1, b, s + 1}, {1, b, s}, Key{1, b, s});
    }
    dataflow("loss-turnaround", {0, b, c.stages - 1}, {1, b, c.stages - 1}, Key{-1, b, c.stages - 1});
  }

  // Kahn's algorithm over contracted nodes.
  std::vector<int> q;
  int live = 0;
  for (int i = 0; i < N; ++i) {
    if (rep[i] != i) continue;
    ++live;
    if (!indeg[i]) q.push_back(i);
  }
  size_t head = 0;
  while (head < q.size()) {
    const int u = q[head++];
    for (int v : out[u])
      if (--indeg[v] == 0) q.push_back(v);
  }
  if (static_cast<int>(q.size()) != live) {
    std::ostringstream os;
    os << "dependency cycle detected; involved actions include:";
    Loc first;
    int shown = 0;
    for (int i = 0; i < N && shown < 4; ++i) {
      if (rep[i] != i || !indeg[i]) continue;
      int d = 0;
      while (base[d + 1] <= i) ++d;
      const Loc x{d, i - base[d]};
      if (first.dev < 0) first = x;
      os << " [device " << x.dev << " pos " << x.pos << " " << describe_action(l.per_device[x.dev][x.pos]) << "]";
      ++shown;
    }
    note(&r, "dependencies", first.dev, first.pos, os.str());
  }
  return r;
}

ValidationReport check_deadlock_free(const ActionList& l) {
  ValidationReport r;
  const int P = static_cast<int>(l.per_device.size());
  const auto groups = exchange_groups(l);

  // Unfused mutual exchanges at adjacent positions on both sides.
  std::map<Key, Loc> tx, rx;
  for (int d = 0; d < P; ++d)
    for (int i = 0; i < static_cast<int>(l.per_device[d].size()); ++i) {
      const Action& a = l.per_device[d][i];
      if (a.kind == ActionKind::Send) tx[outgoing_key(a)] = {d, i};
      if (a.kind == ActionKind::Receive) rx[outgoing_key(a)] = {d, i};
    }
  for (int d = 0; d < P; ++d) {
    const auto& st = l.per_device[d];
    for (int i = 0; i + 1 < static_cast<int>(st.size()); ++i) {
      const Action& x = st[i];
      const Action& y = st[i + 1];
      const bool opp = (x.kind == ActionKind::Send && y.kind == ActionKind::Receive) ||
                       (x.kind == ActionKind::Receive && y.kind == ActionKind::Send);
      if (!opp || x.peer != y.peer || x.peer < 0 || x.peer == d || x.peer < d) continue;
      const Action& s = x.kind == ActionKind::Send ? x : y;
      const Action& v = x.kind == ActionKind::Send ? y : x;
      auto pr = rx.find(outgoing_key(s));
      auto ps = tx.find(outgoing_key(v));
      if (pr == rx.end() || ps == tx.end()) continue;
      if (pr->second.dev != x.peer || ps->second.dev != x.peer) continue;
      if (std::abs(pr->second.pos - ps->second.pos) != 1) continue;
      note(&r, "deadlock_free", d, i,
           "mutual exchange with device " + std::to_string(x.peer) +
               " at adjacent positions on both devices must be fused into a batched exchange");
    }
  }

  // Buffered-send replay.
  std::vector<int> pc(P, 0);
  std::set<std::tuple<int, int, Key>> issued;  // (src, dst, key)
  for (bool moved = true; moved;) {
    moved = false;
    for (int d = 0; d < P; ++d) {
      const auto& st = l.per_device[d];
      while (pc[d] < static_cast<int>(st.size())) {
        const Action& a = st[pc[d]];
        if (a.is_compute() || a.kind == ActionKind::OptimizerStep) {
          // no communication
        } else if (a.kind == ActionKind::Send) {
          if (a.peer < 0 || a.peer >= P || a.peer == d) break;
          issued.insert({d, a.peer, outgoing_key(a)});
        } else if (a.kind == ActionKind::BatchedExchange) {
          auto it = groups.find(a.batch_group);
          if (it == groups.end() || it->second.size() != 2) break;
          const Loc o = other_end(it->second, Loc{d, pc[d]});
          if (o.dev == d || pc[o.dev] != o.pos) break;
          const Action& b = l.per_device[o.dev][o.pos];
          issued.insert({d, a.peer, outgoing_key(a)});
          issued.insert({o.dev, b.peer, outgoing_key(b)});
          ++pc[o.dev];
        } else {  // Receive
          if (a.peer < 0 || a.peer >= P || a.peer == d) break;
          if (!issued.count({a.peer, d, outgoing_key(a)})) break;
        }
        ++pc[d];
        moved = true;
      }
    }
  }
  for (int d = 0; d < P; ++d) {
    if (pc[d] < static_cast<int>(l.per_device[d].size())) {
      note(&r, "deadlock_free", d, pc[d],
           "blocked at " + describe_action(l.per_device[d][pc[d]]) + "; its counterpart is never reached");
    }
  }
  return r;
}

ValidationReport check_flush(const ActionList& l) {
  ValidationReport r;
  for (int d = 0; d < static_cast<int>(l.per_device.size()); ++d) {
    const auto& st = l.per_device[d];
    int first = -1;
    for (int i = 0; i < static_cast<int>(st.size()); ++i) {
      if (st[i].kind != ActionKind::OptimizerStep) continue;
      if (first < 0) first = i;
      else note(&r, "flush", d, i, "duplicate optimizer step");
    }
    if (first < 0) {
      note(&r, "flush", d, -1, "missing flush: no optimizer step");
    } else if (first != static_cast<int>(st.size()) - 1) {
      note(&r, "flush", d, first,
           "premature optimizer step: " + std::to_string(static_cast<int>(st.size()) - 1 - first) +
               " action(s) follow the flush");
    }
  }
  return r;
}

ValidationReport validate_all(const ActionList& l) {
  ValidationReport r = check_completeness(l);
  r.merge(check_dependencies(l));
  r.merge(check_deadlock_free(l));
  r.merge(check_flush(l));
  return r;
}

std::string render_diagnostics_text(const ValidationReport& r) {
  std::string o;
  for (const Diagnostic& d : r.diagnostics) {
    o += d.severity + " [" + d.check + "]";
    if (d.device >= 0) o += " device " + std::to_string(d.device);
    if (d.position >= 0) o += " pos " + std::to_string(d.position);
    o += ": " + d.message + "\n";
  }
  return o;
}

std::string render_diagnostics_json(const ValidationReport& r) {
  auto esc = [](const std::string& s) {
    std::string o;
    for (char ch : s) {
      if (ch == '"' || ch == '\\') o += '\\';
      o += ch;
    }
    return o;
  };
  if (r.diagnostics.empty()) return "[]\n";
  std::string o = "[";
  for (size_t i = 0; i < r.diagnostics.size(); ++i) {
    const Diagnostic& d = r.diagnostics[i];
    o += i ? ",\n  {" : "\n  {";
    o += "\n    \"check\": \"" + esc(d.check) + "\",\n    \"severity\": \"" + esc(d.severity) + "\",";
    o += "\n    \"device\": " + (d.device >= 0 ? std::to_string(d.device) : std::string("null")) + ",";
    o += "\n    \"position\": " + (d.position >= 0 ? std::to_string(d.position) : std::string("null")) + ",";
    o += "\n    \"message\": \"" + esc(d.message) + "\"\n  }";
  }
  return o + "\n]\n";
}

}  // namespace wavepipe
