// Schedule IR: names, configuration, ownership lookup and placements.
//
// Parity notes (reference file:line that each definition must agree with):
//   make_config           src/config.cpp:47-81   (S = 2WP for wave schemes, :79)
//   microbatch_direction  src/action.cpp:85-89
//   slice_owner           src/action.cpp:91-102 (first match in device, rank order)
//   placement_hanayo      src/placement.cpp:52-68 (down 2wP+p, up 2wP+2P-1-p)
#include <array>

#include "wavepipe/core.hpp"

namespace wavepipe {

namespace {

constexpr std::array<const char*, 5> kSchemeNames = {"gpipe", "dapple", "chimera",
                                                     "chimera-wave", "hanayo"};
constexpr std::array<const char*, 6> kKindNames = {"forward", "backward", "send",
                                                   "receive", "batched_exchange",
                                                   "optimizer_step"};

template <typename E, size_t N>
bool lookup(const std::array<const char*, N>& names, const std::string& s, E* out) {
  for (size_t i = 0; i < N; ++i) {
    if (s == names[i]) {
      *out = static_cast<E>(i);
      return true;
    }
  }
  return false;
}

}  // namespace

const char* scheme_name(Scheme s) {
  const auto i = static_cast<size_t>(s);
  return i < kSchemeNames.size() ? kSchemeNames[i] : "?";
}
bool scheme_from_name(const std::string& name, Scheme* out) {
  return lookup(kSchemeNames, name, out);
}
const char* action_kind_name(ActionKind k) {
  const auto i = static_cast<size_t>(k);
  return i < kKindNames.size() ? kKindNames[i] : "?";
}
bool action_kind_from_name(const std::string& name, ActionKind* out) {
  return lookup(kKindNames, name, out);
}
const char* payload_name(Payload p) { return p == Payload::Activation ? "activation" : "gradient"; }
bool payload_from_name(const std::string& name, Payload* out) {
  if (name != "activation" && name != "gradient") return false;
  *out = name == "activation" ? Payload::Activation : Payload::Gradient;
  return true;
}
const char* direction_name(Direction d) { return d == Direction::Down ? "down" : "up"; }
bool direction_from_name(const std::string& name, Direction* out) {
  if (name != "down" && name != "up") return false;
  *out = name == "down" ? Direction::Down : Direction::Up;
  return true;
}

ScheduleConfig make_config(Scheme scheme, int P, int B, int W, int D) {
  auto need = [](bool ok, const std::string& msg) {
    if (!ok) throw ConfigError(msg);
  };
  need(P >= 1, "P must be positive");
  need(B >= 1, "B must be positive");
  need(W >= 1, "W must be positive");
  need(D >= 1, "D must be positive");
  need(B >= P, "B must be >= P: " + std::to_string(B) + " microbatches underfill a " +
                   std::to_string(P) + "-device pipeline");
  const std::string name = scheme_name(scheme);
  if (scheme == Scheme::Chimera || scheme == Scheme::ChimeraWave) {
    need(P % 2 == 0, name + ": P must be even, got " + std::to_string(P));
    need(B % 2 == 0, name + ": B must be even, got " + std::to_string(B));
  }
  need(is_wave_scheme(scheme) || W == 1, name + " does not take waves; W must be 1");
  ScheduleConfig c;
  c.scheme = scheme;
  c.devices = P;
  c.microbatches = B;
  c.waves = W;
  c.replicas = D;
  c.stages = is_wave_scheme(scheme) ? 2 * W * P : P;
  return c;
}

Direction microbatch_direction(const ScheduleConfig& cfg, int mb) {
  // Only Chimera splits the batch: the first ceil(B/2) go down.
  if (cfg.scheme == Scheme::Chimera && mb >= (cfg.microbatches + 1) / 2) return Direction::Up;
  return Direction::Down;
}

SliceOwner slice_owner(const ScheduleConfig& cfg, const StagePlacement& pl, int slice,
                       Direction dir) {
  const bool by_direction = cfg.scheme == Scheme::Chimera;
  for (int d = 0; d < pl.device_count(); ++d) {
    const auto& list = pl.assignment[d];
    for (int r = 0; r < static_cast<int>(list.size()); ++r) {
      if (list[r].index == slice && (!by_direction || list[r].direction == dir)) {
        return SliceOwner{d, r};
      }
    }
  }
  return SliceOwner{};
}

std::string describe_action(const Action& a) {
  std::string s = action_kind_name(a.kind);
  auto field = [&s](const char* name, int v) {
    if (v >= 0) s += std::string(" ") + name + " " + std::to_string(v);
  };
  field("microbatch", a.microbatch);
  field("slice", a.slice_index);
  if (a.payload >= 0) s += std::string(" ") + payload_name(static_cast<Payload>(a.payload));
  field("peer", a.peer);
  field("group", a.batch_group);
  return s;
}

// ---------------------------------------------------------------------------
// Placements.

StagePlacement placement_gpipe(const ScheduleConfig& cfg) {
  StagePlacement pl;
  pl.assignment.resize(cfg.devices);
  for (int p = 0; p < cfg.devices; ++p) pl.assignment[p] = {StageSlice{p, Rational(1), Direction::Down}};
  return pl;
}

StagePlacement placement_dapple(const ScheduleConfig& cfg) { return placement_gpipe(cfg); }

StagePlacement placement_chimera(const ScheduleConfig& cfg) {
  StagePlacement pl;
  pl.assignment.resize(cfg.devices);
  for (int p = 0; p < cfg.devices; ++p) {
    pl.assignment[p] = {StageSlice{p, Rational(1), Direction::Down},
                        StageSlice{cfg.devices - 1 - p, Rational(1), Direction::Up}};
  }
  return pl;
}

StagePlacement placement_hanayo(const ScheduleConfig& cfg) {
  // Wave w occupies global slices [2wP, 2wP+2P): the microbatch walks down the
  // device array on the first P of them and back up on the second P.
  const int P = cfg.devices;
  const Rational share(1, 2 * cfg.waves);
  StagePlacement pl;
  pl.assignment.assign(P, {});
  for (int p = 0; p < P; ++p) {
    for (int w = 0; w < cfg.waves; ++w) {
      const int base = 2 * w * P;
      pl.assignment[p].push_back(StageSlice{base + p, share, Direction::Down});
      pl.assignment[p].push_back(StageSlice{base + 2 * P - 1 - p, share, Direction::Up});
    }
  }
  return pl;
}

StagePlacement make_placement(const ScheduleConfig& cfg) {
  switch (cfg.scheme) {
    case Scheme::GPipe: return placement_gpipe(cfg);
    case Scheme::Dapple: return placement_dapple(cfg);
    case Scheme::Chimera: return placement_chimera(cfg);
    case Scheme::ChimeraWave:
    case Scheme::Hanayo: return placement_hanayo(cfg);
  }
  throw ConfigError("unknown scheme");
}

std::pair<ScheduleConfig, StagePlacement> transform_chimera_to_wave(const ScheduleConfig& cfg) {
  // Ref src/placement.cpp:85-99: the two Chimera replicas fold into two
  // identical one-wave groups of P/2 devices paired as data parallelism.
  if (cfg.scheme != Scheme::Chimera) {
    throw ConfigError("transform_chimera_to_wave requires a chimera config");
  }
  ScheduleConfig w = make_config(Scheme::Hanayo, cfg.devices / 2, cfg.microbatches / 2, 1,
                                 2 * cfg.replicas);
  return {w, placement_hanayo(w)};
}

}  // namespace wavepipe
