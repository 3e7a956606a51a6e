// wavepipe-b200 -- C++ API of the schedule path.
//
// Drop-in for the reference's `namespace wavepipe` headers
// (/root/reference/proj/include/wavepipe/{rational,config,action,cost_model,
// placement,schedule,simulate,analytics}.hpp): the same type names, field
// order, enum values and free-function signatures, so code written against the
// reference compiles unchanged against this library.  The per-header include
// names are kept as thin forwarding headers next to this file.
//
// Everything here is pure host code: immutable value types and re-entrant
// functions (reference SPEC.md:104).  The GPU runtime that *executes* an
// ActionList lives in wavepipe/runtime.hpp.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace wavepipe {

// ---------------------------------------------------------------------------
// Exact fractions (ref include/wavepipe/rational.hpp:29-101).  Always reduced,
// denominator positive, zero is 0/1.
class Rational {
 public:
  constexpr Rational() : n_(0), d_(1) {}
  constexpr Rational(int64_t n) : n_(n), d_(1) {}  // NOLINT: implicit on purpose
  Rational(int64_t n, int64_t d) : n_(n), d_(d) { reduce(); }

  int64_t num() const { return n_; }
  int64_t den() const { return d_; }
  double to_double() const { return double(n_) / double(d_); }
  std::string to_string() const {
    return d_ == 1 ? std::to_string(n_) : std::to_string(n_) + "/" + std::to_string(d_);
  }

  friend Rational operator+(const Rational& x, const Rational& y) {
    const int64_t g = std::gcd(x.d_, y.d_);
    return Rational(x.n_ * (y.d_ / g) + y.n_ * (x.d_ / g), (x.d_ / g) * y.d_);
  }
  friend Rational operator-(const Rational& x, const Rational& y) { return x + (-y); }
  friend Rational operator*(const Rational& x, const Rational& y) {
    const int64_t g1 = std::gcd(x.n_ < 0 ? -x.n_ : x.n_, y.d_);
    const int64_t g2 = std::gcd(y.n_ < 0 ? -y.n_ : y.n_, x.d_);
    return Rational((x.n_ / g1) * (y.n_ / g2), (x.d_ / g2) * (y.d_ / g1));
  }
  friend Rational operator/(const Rational& x, const Rational& y) {
    return x * Rational(y.d_, y.n_);
  }
  Rational operator-() const { Rational r; r.n_ = -n_; r.d_ = d_; return r; }
  Rational& operator+=(const Rational& o) { return *this = *this + o; }
  Rational& operator-=(const Rational& o) { return *this = *this - o; }
  Rational& operator*=(const Rational& o) { return *this = *this * o; }
  Rational& operator/=(const Rational& o) { return *this = *this / o; }

  friend bool operator==(const Rational& x, const Rational& y) { return x.n_ == y.n_ && x.d_ == y.d_; }
  friend bool operator!=(const Rational& x, const Rational& y) { return !(x == y); }
  friend bool operator<(const Rational& x, const Rational& y) {
    return static_cast<__int128>(x.n_) * y.d_ < static_cast<__int128>(y.n_) * x.d_;
  }
  friend bool operator>(const Rational& x, const Rational& y) { return y < x; }
  friend bool operator<=(const Rational& x, const Rational& y) { return !(y < x); }
  friend bool operator>=(const Rational& x, const Rational& y) { return !(x < y); }

 private:
  void reduce() {
    if (d_ == 0) throw std::invalid_argument("Rational: zero denominator");
    if (d_ < 0) { n_ = -n_; d_ = -d_; }
    const int64_t g = std::gcd(n_ < 0 ? -n_ : n_, d_);
    if (g > 1) { n_ /= g; d_ /= g; }
    if (n_ == 0) d_ = 1;
  }
  int64_t n_, d_;
};

// ---------------------------------------------------------------------------
// Schedule configuration (ref include/wavepipe/config.hpp:34-67).
enum class Scheme { GPipe, Dapple, Chimera, ChimeraWave, Hanayo };

const char* scheme_name(Scheme s);
bool scheme_from_name(const std::string& name, Scheme* out);
inline bool is_wave_scheme(Scheme s) { return s == Scheme::Hanayo || s == Scheme::ChimeraWave; }

struct ConfigError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

struct ScheduleConfig {
  Scheme scheme = Scheme::GPipe;
  int devices = 1;       // P
  int microbatches = 1;  // B
  int waves = 1;         // W
  int replicas = 1;      // D (bookkeeping only)
  int stages = 1;        // S = 2WP for wave schemes, else P
};

ScheduleConfig make_config(Scheme scheme, int devices, int microbatches,
                           int waves = 1, int replicas = 1);

// ---------------------------------------------------------------------------
// Action IR (ref include/wavepipe/action.hpp:28-118).
enum class Direction { Down, Up };

struct StageSlice {
  int index = 0;
  Rational fraction{1, 1};
  Direction direction = Direction::Down;
};

struct StagePlacement {
  std::vector<std::vector<StageSlice>> assignment;  // [device][local_module_rank]
  int device_count() const { return static_cast<int>(assignment.size()); }
};

enum class ActionKind { Forward, Backward, Send, Receive, BatchedExchange, OptimizerStep };
enum class Payload { Activation, Gradient };

const char* action_kind_name(ActionKind k);
bool action_kind_from_name(const std::string& name, ActionKind* out);
const char* payload_name(Payload p);
bool payload_from_name(const std::string& name, Payload* out);
const char* direction_name(Direction d);
bool direction_from_name(const std::string& name, Direction* out);

// Seven ints, C-layout compatible with `wp_action` in wavepipe.h.
struct Action {
  ActionKind kind = ActionKind::Forward;
  int microbatch = -1;
  int local_module_rank = -1;
  int slice_index = -1;
  int peer = -1;
  int payload = -1;
  int batch_group = -1;

  bool is_compute() const { return kind == ActionKind::Forward || kind == ActionKind::Backward; }
  bool is_comm() const {
    return kind == ActionKind::Send || kind == ActionKind::Receive ||
           kind == ActionKind::BatchedExchange;
  }
};

struct ActionList {
  ScheduleConfig config;
  StagePlacement placement;
  std::vector<std::vector<Action>> per_device;
};

struct SliceOwner {
  int device = -1;
  int local_rank = -1;
};

Direction microbatch_direction(const ScheduleConfig& cfg, int microbatch);
SliceOwner slice_owner(const ScheduleConfig& cfg, const StagePlacement& placement,
                       int slice_index, Direction dir);
std::string describe_action(const Action& a);

// ---------------------------------------------------------------------------
// Abstract cost model (ref include/wavepipe/cost_model.hpp:27-49).
struct CostModel {
  double t_forward = 1.0;
  double t_backward = 2.0;
  double t_comm = 0.0;

  double slice_forward(const ScheduleConfig& c) const {
    return is_wave_scheme(c.scheme) ? t_forward / (2.0 * c.waves) : t_forward;
  }
  double slice_backward(const ScheduleConfig& c) const {
    return is_wave_scheme(c.scheme) ? t_backward / (2.0 * c.waves) : t_backward;
  }
  CostModel rescaled(int budget_devices, int config_devices) const {
    const double k = static_cast<double>(budget_devices) / config_devices;
    CostModel r = *this;
    r.t_forward *= k;
    r.t_backward *= k;
    return r;
  }
};

// ---------------------------------------------------------------------------
// Placement (ref include/wavepipe/placement.hpp:27-49).
StagePlacement placement_gpipe(const ScheduleConfig& cfg);
StagePlacement placement_dapple(const ScheduleConfig& cfg);
StagePlacement placement_chimera(const ScheduleConfig& cfg);
StagePlacement placement_hanayo(const ScheduleConfig& cfg);
StagePlacement make_placement(const ScheduleConfig& cfg);
std::pair<ScheduleConfig, StagePlacement> transform_chimera_to_wave(const ScheduleConfig& cfg);

// ---------------------------------------------------------------------------
// Schedule generation (ref include/wavepipe/schedule.hpp:26-59).
struct ScheduleError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

ActionList generate_schedule(const StagePlacement& placement, const ScheduleConfig& cfg,
                             const CostModel& cost);
ActionList insert_comm(const ActionList& compute_only);

// ---------------------------------------------------------------------------
// Abstract-time executor (ref include/wavepipe/simulate.hpp:28-80).  The GPU
// runtime fills the same SimTrace with measured seconds.
struct SimulationError : std::runtime_error {
  explicit SimulationError(const std::string& w) : std::runtime_error(w) {}
};

struct TraceInterval {
  int action_index = -1;
  ActionKind kind = ActionKind::Forward;
  int microbatch = -1;
  int slice_index = -1;
  Direction direction = Direction::Down;
  double start = 0.0;
  double end = 0.0;
};

struct CommEvent {
  int src_device = -1;
  int dst_device = -1;
  double post_time = 0.0;
  double arrival_time = 0.0;
};

struct SimTrace {
  double makespan = 0.0;
  std::vector<std::vector<TraceInterval>> intervals;
  std::vector<CommEvent> comm_events;
};

SimTrace simulate(const ActionList& list, const CostModel& cost);
std::string trace_to_json(const SimTrace& trace);
// ref include/wavepipe/gantt.hpp:32 -- "svg" or "csv"; std::invalid_argument otherwise.
std::string trace_to_gantt(const SimTrace& trace, const std::string& format);

// ---------------------------------------------------------------------------
// Analytics (ref include/wavepipe/analytics.hpp:35-140, hot-path subset plus
// the small closed forms).
struct MemoryProfile {
  std::vector<Rational> weight_units;
  std::vector<Rational> peak_activation_units;
};

double bubble_ratio(const SimTrace& trace);
MemoryProfile memory_profile(const SimTrace& trace, const ActionList& list);
Rational activation_variance(const MemoryProfile& profile);

struct ZoneBubbleInput {
  int devices = 1;
  int waves = 1;
  int local_rank = 0;
  double t_forward = 1.0;
  double t_backward = 2.0;
  double t_comm = 0.0;
};
struct ZoneBubbles {
  double a = 0.0;
  double b = 0.0;
  double c_first = 0.0;
  double c_second = 0.0;
};
ZoneBubbles zone_bubbles(const ZoneBubbleInput& input);

Rational analytic_bubble_hanayo(int devices, int waves, const Rational& t_forward,
                                const Rational& t_backward, const Rational& t_comm);
double analytic_bubble_hanayo_d(int devices, int waves, double t_forward,
                                double t_backward, double t_comm);
Rational analytic_bubble_simplified(int devices, int waves);
double analytic_chimera_k(int devices);

struct MetricsReport {
  double makespan = 0.0;
  double bubble_ratio = 0.0;
  std::vector<double> busy;
  MemoryProfile memory;
  Rational activation_variance;
};
MetricsReport compute_metrics(const SimTrace& trace, const ActionList& list);
std::string metrics_to_text(const MetricsReport& report);
std::string metrics_to_json(const MetricsReport& report);

// Scheme comparison sweep (ref include/wavepipe/analytics.hpp:104-140,
// src/analytics.cpp:221-331): every request evaluated at one device budget
// and total microbatch count (chimera-wave as one of its two symmetric
// device groups: half the budget and microbatches, costs rescaled), rows in
// ascending makespan; failures are captured per row and sort last.
struct CompareRequest {
  Scheme scheme = Scheme::GPipe;
  int waves = 1;
};
struct CompareRow {
  Scheme scheme = Scheme::GPipe;
  int devices = 0;       // shared device budget
  int microbatches = 0;  // total microbatches
  int waves = 1;
  double makespan = 0.0;
  double simulated_ratio = 0.0;
  bool has_analytic = false;
  double analytic_ratio = 0.0;
  Rational weight_units;     // per device (max over devices)
  Rational peak_activation;  // max across devices
  Rational variance;
  bool failed = false;
  std::string error;
};
std::vector<CompareRow> compare(const std::vector<CompareRequest>& requests, int budget_devices, int microbatches,
                                const CostModel& base_cost);
// The same rows from MEASURED traces (the GPU runtime's train_step, one per
// request, traces[i] of lists[i]): makespan = measured step (seconds),
// simulated_ratio = bubble_ratio of the measured trace; Hanayo's analytic
// ratio at the measured mean slice costs and the given (measured) message
// latency t_comm.  Same order and writers.
std::vector<CompareRow> compare_measured(const std::vector<CompareRequest>& requests, int budget_devices,
                                         int microbatches, const std::vector<SimTrace>& traces,
                                         const std::vector<ActionList>& lists, double t_comm = 0.0);
std::string compare_to_csv(const std::vector<CompareRow>& rows);
std::string compare_to_json(const std::vector<CompareRow>& rows);

// ---------------------------------------------------------------------------
// Action-list JSON (ref include/wavepipe/serialize.hpp:26-47): stock
// nlohmann-style `dump(2)` bytes, strict parser.
struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
std::string serialize_action_list(const ActionList& list);
ActionList parse_action_list(const std::string& text);

// ---------------------------------------------------------------------------
// Structural validation (ref include/wavepipe/validate.hpp:26-77): run once
// per schedule before the runtime executes it.
struct Diagnostic {
  std::string check;
  std::string severity;
  int device = -1;
  int position = -1;
  std::string message;
};
struct ValidationReport {
  std::vector<Diagnostic> diagnostics;
  bool ok() const { return diagnostics.empty(); }
  void merge(const ValidationReport& o) {
    diagnostics.insert(diagnostics.end(), o.diagnostics.begin(), o.diagnostics.end());
  }
};
ValidationReport check_completeness(const ActionList& list);
ValidationReport check_dependencies(const ActionList& list);
ValidationReport check_deadlock_free(const ActionList& list);
ValidationReport check_flush(const ActionList& list);
ValidationReport validate_all(const ActionList& list);
std::string render_diagnostics_text(const ValidationReport& report);
std::string render_diagnostics_json(const ValidationReport& report);

}  // namespace wavepipe
