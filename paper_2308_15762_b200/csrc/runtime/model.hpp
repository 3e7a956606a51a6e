// Model description for the stage compute: a GPT-like (causal LM) or
// BERT-like (bidirectional, labels on every position) pre-LN decoder stack,
// cut into "units" that the slices of a Hanayo placement partition.
//
// The reference has no model: its slices are abstract shares
// 1/(2W) of a stage (include/wavepipe/action.hpp:34-37,
// src/placement.cpp:52-68).  Here slice s of the S = 2WP slices executes a
// contiguous run of units chosen to balance forward FLOPs, because the
// reference cost model assumes uniform slice cost (cost_model.hpp:32-37).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "wavepipe.h"

namespace wprt {

enum class UnitKind { Embed, Attn, Mlp, Head };

struct Unit {
  UnitKind kind;
  int layer;    // -1 for Embed / Head
  double cost;  // forward FLOPs per token (partition weight)
};

struct ParamDesc {
  std::string name;
  std::vector<int64_t> shape;
  int64_t numel = 0;
  int unit = -1;        // owning unit
  float init_std = 0;   // > 0: N(0, std); else constant init_value
  float init_value = 0;
};

struct ModelSpec {
  int layers, hidden, heads, ffn, seq, vocab, mbs;
  bool causal, tie;
  int dtype;  // wpk::kF32 / wpk::kBF16
  int optimizer;
  float lr, beta1, beta2, eps, weight_decay;
  uint64_t seed;

  static ModelSpec from_desc(const wp_model_desc& d);
  int tokens() const { return mbs * seq; }  // T per microbatch
  int head_dim() const { return hidden / heads; }
  int act_bytes() const { return dtype == 0 ? 4 : 2; }
};

std::vector<Unit> build_units(const ModelSpec& m);

// Contiguous partition of units into S slices: bounds[k]..bounds[k+1]-1 run in
// slice k.  Cuts go where the cumulative forward cost is closest to k/S of
// the total; the embedding always lands in slice 0 and the LM head in slice
// S-1 (so tied embeddings stay on one Hanayo device); slices may be empty
// (identity) when S exceeds the unit count.
std::vector<int> partition_units(const std::vector<Unit>& units, int S);

// Device-balanced variant used by the runtime: slice k runs on pipeline
// device slice_device[k] (the placement), and the cuts minimise the busiest
// device's total cost (a synchronous flush step is bounded by it) rather
// than equalising slices -- the LM head alone is ~2 layers of GPT-1.3B, so
// equal slices leave the head's device (Hanayo device 0) 1.5x loaded at
// P=8 W=2; balanced devices bring it to ~1.1x.
std::vector<int> partition_units(const std::vector<Unit>& units, const std::vector<int>& slice_device, int P);

// Parameters of one unit, in a fixed order (names are global, layer-indexed).
std::vector<ParamDesc> unit_params(const ModelSpec& m, int unit_index, const Unit& u);

}  // namespace wprt
