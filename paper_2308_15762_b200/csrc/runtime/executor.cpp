// Runtime: parameters, stash pools and the per-device action interpreter.
// See runtime.hpp for the executor contract and its reference citations.
#include <cuda_bf16.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <thread>

#include <nvtx3/nvToolsExt.h>

#include "capi_internal.hpp"
#include "kernels/attention.cuh"
#include "runtime/device_state.hpp"
#include "runtime/runtime.hpp"
#include "runtime/stream_ops.hpp"

namespace wprt {

using wavepipe::Action;
using wavepipe::ActionKind;

namespace {

constexpr int kAct = static_cast<int>(wavepipe::Payload::Activation);
constexpr int kGrad = static_cast<int>(wavepipe::Payload::Gradient);


uint64_t name_hash(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

}  // namespace

// --------------------------------------------------------------------- pool
Pool::~Pool() {
  if (leak_) return;
  DevGuard g(dev_);
  for (auto& b : all_) {
    if (b->p) cudaFree(b->p);
    if (b->ev) cudaEventDestroy(b->ev);
  }
}

BufPtr Pool::alloc(size_t bytes, cudaStream_t stream, int cls) {
  bytes = (bytes + 255) & ~size_t(255);
  auto& fl = free_[{cls, bytes}];
  // Reuse a buffer only if that adds no wait on another stream's pending
  // work: a message buffer freed by a push on a copy stream is busy until
  // the receiver posts it, and making the compute stream wait for that
  // would turn the reference's buffered sends (src/simulate.cpp:117-122)
  // into blocking ones -- a cross-device wait the action list does not have
  // (it deadlocks Chimera P=4).  Such buffers are skipped and the pool grows
  // by the messages in flight instead.
  for (size_t i = fl.size(); i-- > 0;) {
    BufPtr b = fl[i];
    if (b->ev_pending && b->released_on != stream) {
      const cudaError_t q = cudaEventQuery(b->ev);
      if (q == cudaErrorNotReady) continue;
      ck(q, "pool event query");
    } else if (b->ev_pending) {
      ck(cudaStreamWaitEvent(stream, b->ev, 0), "pool wait");  // same stream: program order, no new wait
    }
    b->ev_pending = false;
    fl.erase(fl.begin() + static_cast<long>(i));
    return b;
  }
  DevGuard g(dev_);
  auto b = std::make_shared<Buf>();
  ck(cudaMalloc(&b->p, bytes), "cudaMalloc (stash pool)");
  b->bytes = bytes;
  b->pool_class = cls;
  reserved_ += bytes;
  all_.push_back(b);
  return b;
}

void Pool::release(const BufPtr& b, cudaStream_t stream) {
  if (!b) return;

  // Message buffers and anything released off the compute stream carry an
  // event: the next owner (possibly another stream or device) waits on it.
  if (b->pool_class == 1 || stream != home_) {
    if (!b->ev) {
      DevGuard g(dev_);
      ck(cudaEventCreateWithFlags(&b->ev, cudaEventDisableTiming), "event create");
    }
    ck(cudaEventRecord(b->ev, stream), "pool release record");
    b->ev_pending = true;
    b->released_on = stream;
  }
  free_[{b->pool_class, b->bytes}].push_back(b);
}


// ------------------------------------------------------------------ runtime
Runtime::Runtime(const wp_model_desc& desc, const wavepipe::ActionList& list, int transport, const int* device_ids,
                 int rank)
    : m_(ModelSpec::from_desc(desc)), list_(list), transport_(transport), rank_(rank) {
  // IPC transport: `rank` is the global rank replica * P + pipeline device.
  replicas_ = std::max(1, list_.config.replicas);
  if (transport_ == WP_TRANSPORT_IPC) {
    if (rank < 0 || rank >= list_.config.devices * replicas_) {
      throw wavepipe::ConfigError("IPC transport needs 0 <= rank < P * D");
    }
    replica_ = rank / list_.config.devices;
    rank_ = rank % list_.config.devices;
  } else if (replicas_ > 1) {
    throw wavepipe::ConfigError("data-parallel replicas (D > 1) need the IPC transport");
  }
  const auto rep = wavepipe::validate_all(list_);
  if (!rep.ok()) {
    throw wavepipe::ScheduleError("action list fails validation:\n" + wavepipe::render_diagnostics_text(rep));
  }
  units_ = build_units(m_);
  {
    std::vector<int> slice_device(list_.config.stages, 0);
    for (int d = 0; d < static_cast<int>(list_.placement.assignment.size()); ++d)
      for (const auto& sl : list_.placement.assignment[d]) slice_device[sl.index] = d;
    bounds_ = partition_units(units_, slice_device, list_.config.devices);
  }
  if (m_.tie) {  // every device holding the embedding slice also holds the head slice (Hanayo, Chimera)
    for (const auto& dev : list_.placement.assignment) {
      bool first = false, last = false;
      for (const auto& sl : dev) first |= sl.index == 0, last |= sl.index == list_.config.stages - 1;
      if (first != last) {
        throw wavepipe::ConfigError(
            "tie_embeddings needs the first and last slice on one device (true for Hanayo and Chimera placements)");
      }
    }
  }
  if (list_.config.scheme == wavepipe::Scheme::Chimera && transport_ != WP_TRANSPORT_IPC) {
    throw wavepipe::ConfigError(
        "Chimera holds every stage on two devices (p and P-1-p) that sum their gradients over peer memory: "
        "it needs the IPC transport (one process per device)");
  }
  if (transport_ != WP_TRANSPORT_LOCAL && transport_ != WP_TRANSPORT_IPC) {
    throw wavepipe::ConfigError(transport_ == 1 ? "transport 1 (NCCL) was removed: use WP_TRANSPORT_IPC"
                                                : "unknown transport");
  }
  if (const char* t = std::getenv("WP_STALL_TIMEOUT_S")) {
    const double v = std::atof(t);
    if (v > 0) stall_timeout_s_ = v;
  }
  build_devices(device_ids);
  if (transport_ == WP_TRANSPORT_IPC) ipc_setup();
}

Runtime::~Runtime() {
  if (broken_ && !released_) {
    // A stalled step whose device waits could not be released: the streams
    // stay blocked until the process exits, and every freeing call below
    // (cudaFree, cudaDeviceSynchronize) would block with them.  Leak the
    // device state instead; the driver reclaims it at process exit.
    for (auto& d : devs_) d->pool->leak();
    for (auto& d : devs_) d.release();
    return;
  }
  ipc_release();
  if (input_ready_) {
    DevGuard g(input_ready_dev_);
    cudaEventDestroy(input_ready_);
  }
  for (auto& d : devs_) {
    DevGuard g(d->cuda);
    cudaDeviceSynchronize();
    for (auto e : d->events) cudaEventDestroy(e);
    if (d->step_begin) cudaEventDestroy(d->step_begin);
    for (void* p : {static_cast<void*>(d->master), static_cast<void*>(d->grad), static_cast<void*>(d->m),
                    static_cast<void*>(d->v), d->shadow, static_cast<void*>(d->loss), static_cast<void*>(d->tokens),
                    static_cast<void*>(d->labels), static_cast<void*>(d->scores),
                    static_cast<void*>(d->attn_delta), static_cast<void*>(d->dq_acc),
                    static_cast<void*>(d->ln_rows)})
      if (p) cudaFree(p);
    d->pool.reset();
    if (d->clock_host) cudaFreeHost(d->clock_host);
    if (d->compute) cudaStreamDestroy(d->compute);
    if (d->copy) cudaStreamDestroy(d->copy);
    for (auto& kv : d->tx) cudaStreamDestroy(kv.second);
  }
}

int Runtime::owner_device(int mb, int slice) const {
  return wavepipe::slice_owner(list_.config, list_.placement, slice,
                               wavepipe::microbatch_direction(list_.config, mb))
      .device;
}

void Runtime::build_devices(const int* device_ids) {
  const int P = list_.config.devices;
  dev_of_pipeline_.assign(P, -1);
  std::vector<int> local;
  if (transport_ == WP_TRANSPORT_LOCAL) {
    for (int p = 0; p < P; ++p) local.push_back(p);
  } else {
    local.push_back(rank_);
  }
  const int B = list_.config.microbatches, T = m_.tokens();
  for (size_t i = 0; i < local.size(); ++i) {
    auto d = std::make_unique<DeviceState>();
    d->pipe = local[i];
    d->cuda = device_ids ? device_ids[transport_ == WP_TRANSPORT_LOCAL ? i : 0] : 0;
    dev_of_pipeline_[d->pipe] = static_cast<int>(i);
    DevGuard g(d->cuda);
    ck(cudaStreamCreateWithFlags(&d->compute, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&d->copy, cudaStreamNonBlocking), "stream");
    d->pool = std::make_unique<Pool>(d->cuda, d->compute);
    ck(cudaEventCreate(&d->step_begin), "event");
    // Parameters of every unit of every slice this device holds.
    std::vector<int> mine;
    for (int s : [&] {
           std::vector<int> v;
           for (const auto& sl : list_.placement.assignment[d->pipe]) v.push_back(sl.index);
           return v;
         }()) {
      for (int u = bounds_[s]; u < bounds_[s + 1]; ++u) mine.push_back(u);
    }
    std::sort(mine.begin(), mine.end());
    int64_t off = 0;
    for (int u : mine) {
      for (auto& pd : unit_params(m_, u, units_[u])) {
        ParamSlot slot;
        slot.desc = pd;
        slot.offset = off;
        off += (pd.numel + 63) / 64 * 64;
        d->by_name[pd.name] = static_cast<int>(d->params.size());
        param_index_[pd.name] = ParamRef{static_cast<int>(i), static_cast<int>(d->params.size()), pd};
        param_names_.push_back(pd.name);
        d->params.push_back(slot);
      }
    }
    d->nparam = std::max<int64_t>(off, 64);
    const size_t pb = d->nparam * sizeof(float);
    ck(cudaMalloc(&d->master, pb), "cudaMalloc params");
    ck(cudaMalloc(&d->grad, pb), "cudaMalloc grads");
    ck(cudaMemset(d->grad, 0, pb), "memset");
    if (m_.optimizer == 1) {
      ck(cudaMalloc(&d->m, pb), "cudaMalloc adam m");
      ck(cudaMalloc(&d->v, pb), "cudaMalloc adam v");
      ck(cudaMemset(d->m, 0, pb), "memset");
      ck(cudaMemset(d->v, 0, pb), "memset");
    }
    if (m_.dtype == wpk::kBF16) ck(cudaMalloc(&d->shadow, d->nparam * 2), "cudaMalloc shadow");
    ck(cudaMalloc(&d->loss, sizeof(float)), "cudaMalloc loss");
    ck(cudaMalloc(&d->tokens, sizeof(int32_t) * B * T), "cudaMalloc tokens");
    ck(cudaMalloc(&d->labels, sizeof(int32_t) * B * T), "cudaMalloc labels");
    ck(cudaMalloc(&d->ln_rows, sizeof(float) * 2 * size_t(T)), "cudaMalloc ln rows");
    if (use_flash()) {
      ck(cudaMalloc(&d->attn_delta, sizeof(float) * size_t(m_.mbs) * m_.heads * m_.seq), "cudaMalloc delta");
      ck(cudaMalloc(&d->dq_acc, sizeof(float) * size_t(T) * m_.hidden), "cudaMalloc dq");
    } else {
      const size_t sc = sizeof(float) * size_t(m_.mbs) * m_.heads * m_.seq * m_.seq;
      ck(cudaMalloc(&d->scores, sc), "cudaMalloc scores");
    }
    init_params(*d);
    ck(cudaDeviceSynchronize(), "init sync");
    devs_.push_back(std::move(d));
  }
  // BE counterparts, resolved once (ref include/wavepipe/action.hpp:67-73).
  std::map<int, std::vector<std::pair<int, int>>> groups;
  for (int p = 0; p < P; ++p)
    for (int i = 0; i < static_cast<int>(list_.per_device[p].size()); ++i)
      if (list_.per_device[p][i].kind == ActionKind::BatchedExchange)
        groups[list_.per_device[p][i].batch_group].push_back({p, i});
  for (auto& d : devs_) d->be_partner.assign(list_.per_device[d->pipe].size(), {-1, -1});
  for (auto& [g, ends] : groups) {
    for (int k = 0; k < 2; ++k) {
      const int li = dev_of_pipeline_[ends[k].first];
      if (li >= 0) devs_[li]->be_partner[ends[k].second] = ends[1 - k];
    }
  }
}

void Runtime::init_params(DeviceState& d) {
  for (auto& s : d.params) {
    float* p = d.master + s.offset;
    if (s.desc.init_std > 0) {
      launches_ += wpk::init_normal(p, s.desc.numel, s.desc.init_std, m_.seed ^ name_hash(s.desc.name), d.compute);
    } else {
      launches_ += wpk::fill_f32(p, s.desc.numel, s.desc.init_value, d.compute);
    }
  }
  if (d.shadow) launches_ += wpk::cast_f32_to_bf16(d.master, d.shadow, d.nparam, d.compute);
}

const void* Runtime::weight(DeviceState& d, const std::string& name) const {
  auto it = d.by_name.find(name);
  if (it == d.by_name.end()) throw std::runtime_error("parameter not on this device: " + name);
  const int64_t off = d.params[it->second].offset;
  if (m_.dtype == wpk::kBF16) return static_cast<const __nv_bfloat16*>(d.shadow) + off;
  return d.master + off;
}

float* Runtime::master(DeviceState& d, const std::string& name) const {
  auto it = d.by_name.find(name);
  if (it == d.by_name.end()) throw std::runtime_error("parameter not on this device: " + name);
  return d.master + d.params[it->second].offset;
}

float* Runtime::grad(DeviceState& d, const std::string& name) const {
  auto it = d.by_name.find(name);
  if (it == d.by_name.end()) throw std::runtime_error("parameter not on this device: " + name);
  return d.grad + d.params[it->second].offset;
}

namespace {

// Debugging aid (WP_DEBUG_CHECK_GEMM=1): recompute sampled outputs of every
// GEMM on the host from the device operands and report the first mismatch.
float host_elem(const std::vector<uint16_t>& h, const std::vector<float>& f, int dtype, int64_t i) {
  if (dtype == wpk::kF32) return f[i];
  uint32_t u = static_cast<uint32_t>(h[i]) << 16;
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}

struct HostBuf {
  std::vector<uint16_t> h;
  std::vector<float> f;
  int dtype;
  void fetch(const void* p, int64_t n, int dt) {
    dtype = dt;
    if (dt == wpk::kF32) {
      f.resize(n);
      cudaMemcpy(f.data(), p, n * 4, cudaMemcpyDeviceToHost);
    } else {
      h.resize(n);
      cudaMemcpy(h.data(), p, n * 2, cudaMemcpyDeviceToHost);
    }
  }
  float at(int64_t i) const { return host_elem(h, f, dtype, i); }
};

int64_t operand_extent(const wpk::Operand& o, int rows, int K, int nb1, int nb2) {
  const int64_t inner = o.mn_major ? static_cast<int64_t>(K - 1) * o.ld + rows : static_cast<int64_t>(rows - 1) * o.ld + K;
  return inner + static_cast<int64_t>(nb1 - 1) * o.b1 + static_cast<int64_t>(nb2 - 1) * o.b2;
}

void check_gemm(const wpk::GemmProblem& g, cudaStream_t s, const std::function<void()>& run) {
  const int cdt = g.epi.mode == wpk::kEpiAccum ? wpk::kF32 : g.epi.c_dtype;
  const int64_t c_ext = static_cast<int64_t>(g.M - 1) * g.epi.ldc + g.N +
                        static_cast<int64_t>(g.nb1 - 1) * g.epi.c_b1 + static_cast<int64_t>(g.nb2 - 1) * g.epi.c_b2;
  cudaStreamSynchronize(s);
  HostBuf A, B, C0, R, X;
  A.fetch(g.A.ptr, operand_extent(g.A, g.M, g.K, g.nb1, g.nb2), g.in_dtype);
  B.fetch(g.B.ptr, operand_extent(g.B, g.N, g.K, g.nb1, g.nb2), g.in_dtype);
  if (g.epi.mode == wpk::kEpiAccum) C0.fetch(g.epi.c, c_ext, cdt);
  if (g.epi.mode == wpk::kEpiResidual) R.fetch(g.epi.resid, c_ext, cdt);
  if (g.epi.mode == wpk::kEpiDGelu) X.fetch(g.epi.aux, c_ext, cdt);
  std::vector<float> bias;
  if (g.epi.bias) {
    bias.resize(g.N);
    cudaMemcpy(bias.data(), g.epi.bias, g.N * 4, cudaMemcpyDeviceToHost);
  }
  run();
  cudaStreamSynchronize(s);
  HostBuf C;
  C.fetch(g.epi.c, c_ext, cdt);
  uint64_t rng = 88172645463325252ull;
  auto rnd = [&](int n) {
    rng ^= rng << 13, rng ^= rng >> 7, rng ^= rng << 17;
    return static_cast<int>(rng % static_cast<uint64_t>(n));
  };
  auto gelu = [](double x) { return 0.5 * x * (1 + std::tanh(0.7978845608028654 * (x + 0.044715 * x * x * x))); };
  auto dgelu = [](double x) {
    const double t = std::tanh(0.7978845608028654 * (x + 0.044715 * x * x * x));
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * x * x);
  };
  const int64_t total = int64_t(g.M) * g.N * g.nb1 * g.nb2;
  const bool full = total * g.K <= 40000000;
  const int64_t iters = full ? total : 4096;
  int64_t bad = 0;
  for (int64_t it = 0; it < iters; ++it) {
    int z1, z2, m, n;
    if (full) {
      int64_t r = it;
      n = static_cast<int>(r % g.N), r /= g.N;
      m = static_cast<int>(r % g.M), r /= g.M;
      z1 = static_cast<int>(r % g.nb1), z2 = static_cast<int>(r / g.nb1);
    } else {
      z1 = rnd(g.nb1), z2 = rnd(g.nb2), m = rnd(g.M), n = rnd(g.N);
    }
    if (g.causal == wpk::kCausalSkipUpper && n > m) continue;
    int k0 = 0, k1 = g.K;
    if (g.causal == wpk::kCausalKUpToRow) k1 = std::min(g.K, (m / 128 + 1) * 128);
    if (g.causal == wpk::kCausalKFromRow) k0 = (m / 128) * 128;
    double acc = 0, mag = 0;
    for (int k = k0; k < k1; ++k) {
      const int64_t ai = z1 * g.A.b1 + z2 * g.A.b2 + (g.A.mn_major ? int64_t(k) * g.A.ld + m : int64_t(m) * g.A.ld + k);
      const int64_t bi = z1 * g.B.b1 + z2 * g.B.b2 + (g.B.mn_major ? int64_t(k) * g.B.ld + n : int64_t(n) * g.B.ld + k);
      const double pr = double(A.at(ai)) * double(B.at(bi));
      acc += pr;
      mag += std::fabs(pr);
    }
    const int64_t ci = z1 * g.epi.c_b1 + z2 * g.epi.c_b2 + int64_t(m) * g.epi.ldc + n;
    double want = acc * g.epi.alpha + (g.epi.bias ? bias[n] : 0.0);
    double tol_scale = mag * std::fabs(g.epi.alpha) + (g.epi.bias ? std::fabs(bias[n]) : 0.0);
    switch (g.epi.mode) {
      case wpk::kEpiAccum: want += C0.at(ci); tol_scale += std::fabs(C0.at(ci)); break;
      case wpk::kEpiResidual: want += R.at(ci); tol_scale += std::fabs(R.at(ci)); break;
      case wpk::kEpiGelu: want = gelu(want); break;
      case wpk::kEpiDGelu: want *= dgelu(X.at(ci)); tol_scale *= 1.2; break;
      default: break;
    }
    const double got = C.at(ci);
    // bf16 x bf16 products are exact in fp32; fp32 accumulation error ~K ulps of
    // sum|p|; a bf16 output adds one rounding (2^-9 relative).
    const double tol = 1e-7 + 2e-5 * tol_scale + (cdt == wpk::kF32 ? 1e-6 : 8e-3) * std::fabs(want);
    if (!(std::fabs(got - want) <= tol) && bad++ < 3) {
      std::fprintf(stderr,
                   "GEMM CHECK FAILED: M=%d N=%d K=%d nb=%dx%d A_mn=%d B_mn=%d mode=%d causal=%d c_dtype=%d at "
                   "z=(%d,%d) m=%d n=%d: got %.6g want %.6g (tol %.3g)\n",
                   g.M, g.N, g.K, g.nb1, g.nb2, int(g.A.mn_major), int(g.B.mn_major), g.epi.mode, g.causal,
                   g.epi.c_dtype, z1, z2, m, n, got, want, tol);
    }
  }
  if (bad) std::fprintf(stderr, "GEMM CHECK: %lld of %lld checked outputs wrong\n", (long long)bad, (long long)iters);
}

bool check_ops_enabled() {
  static const bool on = std::getenv("WP_DEBUG_CHECK_OPS") != nullptr;  // debugging aid
  return on;
}

void report(const char* what, int64_t bad, int64_t n, double worst) {
  if (bad) std::fprintf(stderr, "OP CHECK %s: %lld of %lld wrong (worst %.3g)\n", what, (long long)bad, (long long)n, worst);
}

void check_layernorm(int dt, const void* x, const float* w, const float* b, const void* y, const float* mean,
                     const float* rstd, int T, int h, cudaStream_t s) {
  cudaStreamSynchronize(s);
  HostBuf X, Y, W, Bb, Mu, Rs;
  X.fetch(x, int64_t(T) * h, dt);
  Y.fetch(y, int64_t(T) * h, dt);
  W.fetch(w, h, wpk::kF32);
  Bb.fetch(b, h, wpk::kF32);
  Mu.fetch(mean, T, wpk::kF32);
  Rs.fetch(rstd, T, wpk::kF32);
  int64_t bad = 0;
  double worst = 0;
  for (int t = 0; t < T; ++t) {
    double mu = 0, var = 0;
    for (int c = 0; c < h; ++c) mu += X.at(int64_t(t) * h + c);
    mu /= h;
    for (int c = 0; c < h; ++c) var += (X.at(int64_t(t) * h + c) - mu) * (X.at(int64_t(t) * h + c) - mu);
    const double rs = 1.0 / std::sqrt(var / h + 1e-5);
    for (int c = 0; c < h; ++c) {
      const double want = (X.at(int64_t(t) * h + c) - mu) * rs * W.at(c) + Bb.at(c);
      const double err = std::fabs(Y.at(int64_t(t) * h + c) - want);
      if (err > 1e-2 * (1 + std::fabs(want))) ++bad, worst = std::max(worst, err);
    }
    if (std::fabs(Mu.at(t) - mu) > 1e-3 * (1 + std::fabs(mu))) ++bad;
  }
  report("layernorm_fwd", bad, int64_t(T) * h, worst);
}

// LayerNorm backward: dx vs host, and the dw/db increments.
struct LnBwdCheck {
  HostBuf DY, X, MU, RS, W, R, DW0, DB0;
  int dt, T, h;
  bool has_res;
  void before(int dt_, const void* dy, const void* x, const float* mean, const float* rstd, const float* w,
              const void* dres, const float* dw, const float* db, int T_, int h_, cudaStream_t s) {
    cudaStreamSynchronize(s);
    dt = dt_, T = T_, h = h_, has_res = dres != nullptr;
    DY.fetch(dy, int64_t(T) * h, dt);
    X.fetch(x, int64_t(T) * h, dt);
    MU.fetch(mean, T, wpk::kF32);
    RS.fetch(rstd, T, wpk::kF32);
    W.fetch(w, h, wpk::kF32);
    if (has_res) R.fetch(dres, int64_t(T) * h, dt);
    DW0.fetch(dw, h, wpk::kF32);
    DB0.fetch(db, h, wpk::kF32);
  }
  void after(const void* dx, const float* dw, const float* db, cudaStream_t s) {
    cudaStreamSynchronize(s);
    HostBuf DX, DW, DB;
    DX.fetch(dx, int64_t(T) * h, dt);
    DW.fetch(dw, h, wpk::kF32);
    DB.fetch(db, h, wpk::kF32);
    std::vector<double> gw(h, 0), gb(h, 0);
    int64_t bad = 0;
    double worst = 0;
    for (int t = 0; t < T; ++t) {
      double sg = 0, sgx = 0;
      for (int c = 0; c < h; ++c) {
        const int64_t i = int64_t(t) * h + c;
        const double xh = (X.at(i) - MU.at(t)) * RS.at(t), g = DY.at(i) * W.at(c);
        sg += g, sgx += g * xh;
        gw[c] += DY.at(i) * xh, gb[c] += DY.at(i);
      }
      sg /= h, sgx /= h;
      for (int c = 0; c < h; ++c) {
        const int64_t i = int64_t(t) * h + c;
        const double xh = (X.at(i) - MU.at(t)) * RS.at(t);
        const double want = RS.at(t) * (DY.at(i) * W.at(c) - sg - xh * sgx) + (has_res ? R.at(i) : 0.0);
        const double err = std::fabs(DX.at(i) - want);
        if (err > 1e-2 * std::fabs(want) + 1e-3 * RS.at(t) * std::fabs(sg) + 1e-7) ++bad, worst = std::max(worst, err);
      }
    }
    report("layernorm_bwd dx", bad, int64_t(T) * h, worst);
    bad = 0, worst = 0;
    for (int c = 0; c < h; ++c) {
      const double ew = std::fabs(DW.at(c) - DW0.at(c) - gw[c]), eb = std::fabs(DB.at(c) - DB0.at(c) - gb[c]);
      if (ew > 1e-4 * std::fabs(gw[c]) + 1e-7 || eb > 1e-4 * std::fabs(gb[c]) + 1e-7) ++bad, worst = std::max(worst, std::max(ew, eb));
    }
    report("layernorm_bwd dw/db", bad, h, worst);
  }
};

void check_softmax(int dt, const float* S, const void* P, int rows, int n, int causal, cudaStream_t s) {
  cudaStreamSynchronize(s);
  HostBuf Sh, Ph;
  Sh.fetch(S, int64_t(rows) * n, wpk::kF32);
  Ph.fetch(P, int64_t(rows) * n, dt);
  int64_t bad = 0;
  double worst = 0;
  for (int r = 0; r < rows; ++r) {
    const int q = r % n, valid = causal ? q + 1 : n;
    double m = -1e300, sum = 0;
    for (int j = 0; j < valid; ++j) m = std::max(m, double(Sh.at(int64_t(r) * n + j)));
    for (int j = 0; j < valid; ++j) sum += std::exp(Sh.at(int64_t(r) * n + j) - m);
    for (int j = 0; j < valid; ++j) {
      const double want = std::exp(Sh.at(int64_t(r) * n + j) - m) / sum;
      const double err = std::fabs(Ph.at(int64_t(r) * n + j) - want);
      if (err > 1e-2 * want + 1e-6) ++bad, worst = std::max(worst, err);
    }
  }
  report("softmax_fwd", bad, int64_t(rows) * n, worst);
}


}  // namespace

void Runtime::gemm(DeviceState& d, const wpk::GemmProblem& g) {
  static const bool check = std::getenv("WP_DEBUG_CHECK_GEMM") != nullptr;  // debugging aid
  if (check) {
    check_gemm(g, d.compute, [&] { launches_ += wpk::gemm(g, d.compute); });
    return;
  }
  static const bool sync_each = std::getenv("WP_DEBUG_SYNC_GEMM") != nullptr;  // debugging aid
  if (sync_each) {
    ck(cudaStreamSynchronize(d.compute), "debug sync");
    launches_ += wpk::gemm(g, d.compute);
    ck(cudaStreamSynchronize(d.compute), "debug sync");
    return;
  }
  if (!profiling_) {
    launches_ += wpk::gemm(g, d.compute);
    return;
  }
  cudaEvent_t s = next_event(d), e = next_event(d);
  ck(cudaEventRecord(s, d.compute), "record gemm start");
  launches_ += wpk::gemm(g, d.compute);
  ck(cudaEventRecord(e, d.compute), "record gemm end");
  const std::string shape = std::to_string(g.M) + "x" + std::to_string(g.N) + "x" + std::to_string(g.K) + " b" +
                            std::to_string(g.nb1 * g.nb2) + " " + (g.A.mn_major ? "M" : "K") +
                            (g.B.mn_major ? "N" : "K") + " c" + std::to_string(g.causal);
  d.gemm_recs.push_back({2.0 * g.M * g.N * g.K * g.nb1 * g.nb2, s, e, shape});
}

template <typename F>
void Runtime::timed_attention(DeviceState& d, bool backward, F&& launch) {
  if (!profiling_) {
    launch();
    return;
  }
  cudaEvent_t s = next_event(d), e = next_event(d);
  ck(cudaEventRecord(s, d.compute), "record attention start");
  launch();
  ck(cudaEventRecord(e, d.compute), "record attention end");
  // algorithmic FLOPs: 4 mbs heads seq^2 d (half when causal); backward 2.5x
  const double fwd = 4.0 * m_.mbs * m_.heads * double(m_.seq) * m_.seq * m_.head_dim() / (m_.causal ? 2.0 : 1.0);
  d.gemm_recs.push_back({backward ? 2.5 * fwd : fwd, s, e, backward ? "flash attention bwd" : "flash attention fwd",
                         true});
}

template <typename F>
void Runtime::timed_hbm(DeviceState& d, const char* cls, double bytes, F&& launch) {
  if (!profiling_) {
    launch();
    return;
  }
  cudaEvent_t s = next_event(d), e = next_event(d);
  ck(cudaEventRecord(s, d.compute), "record hbm start");
  launch();
  ck(cudaEventRecord(e, d.compute), "record hbm end");
  DeviceState::GemmRec r{bytes, s, e, cls};
  r.hbm = true;
  d.gemm_recs.push_back(r);
}

bool Runtime::use_flash() const {
  static const bool off = std::getenv("WP_NO_FLASH") != nullptr;
  return !off && m_.dtype == wpk::kBF16 && wpk::flash_supported(attn_shape());
}

wpk::AttnShape Runtime::attn_shape() const {
  return wpk::AttnShape{m_.mbs, m_.seq, m_.heads, m_.head_dim(), m_.hidden, m_.causal ? 1 : 0};
}

cudaEvent_t Runtime::next_event(DeviceState& d) {
  if (d.ev_next == d.events.size()) {
    DevGuard g(d.cuda);
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "event create");
    d.events.push_back(e);
  }
  return d.events[d.ev_next++];
}

// ------------------------------------------------------------ unit kernels
namespace {

wpk::Operand op(const void* p, int64_t ld, bool mn, int64_t b1 = 0, int64_t b2 = 0) {
  return wpk::Operand{p, ld, mn, b1, b2};
}

void* at(const BufPtr& b, int64_t elems, int es) { return static_cast<char*>(b->p) + elems * es; }

}  // namespace

BufPtr Runtime::unit_fwd(DeviceState& d, int ui, int mb, BufPtr x, UnitStash& st) {
  const Unit& u = units_[ui];
  const int T = m_.tokens(), h = m_.hidden, f = m_.ffn, V = m_.vocab, S = m_.seq, H = m_.heads, dh = m_.head_dim();
  const int es = m_.act_bytes(), dt = m_.dtype;
  cudaStream_t cs = d.compute;
  Pool& pool = *d.pool;
  auto act = [&](int64_t n) { return pool.alloc(n * es, cs, 0); };
  auto f32 = [&](int64_t n) { return pool.alloc(n * 4, cs, 0); };
  const std::string L = "h." + std::to_string(u.layer) + ".";

  if (u.kind == UnitKind::Embed) {
    BufPtr out = act(int64_t(T) * h);
    // tokens, the T gathered wte rows, the wpe table, the output
    timed_hbm(d, "embedding_fwd", 4.0 * T + double(es) * (2.0 * T * h + double(S) * h), [&] {
      launches_ += wpk::embed_fwd(dt, d.tokens + int64_t(mb) * T, weight(d, "wte"), weight(d, "wpe"), out->p, T, S,
                                  h, cs);
    });
    return out;
  }
  st.x = x;
  st.ln = act(int64_t(T) * h);
  st.mean = f32(T);
  st.rstd = f32(T);
  const char* lnw = u.kind == UnitKind::Attn ? "ln1" : u.kind == UnitKind::Mlp ? "ln2" : nullptr;
  const std::string lnname = u.kind == UnitKind::Head ? "lnf" : L + lnw;
  // x in, y out, mean / rstd out, w / b in
  timed_hbm(d, "layernorm_fwd", 2.0 * es * T * h + 8.0 * T + 8.0 * h, [&] {
    launches_ += wpk::layernorm_fwd(dt, x->p, master(d, lnname + ".w"), master(d, lnname + ".b"), st.ln->p,
                                    static_cast<float*>(st.mean->p), static_cast<float*>(st.rstd->p), T, h, cs);
  });
  if (check_ops_enabled())
    check_layernorm(dt, x->p, master(d, lnname + ".w"), master(d, lnname + ".b"), st.ln->p,
                    static_cast<float*>(st.mean->p), static_cast<float*>(st.rstd->p), T, h, cs);
  wpk::GemmProblem g;
  g.in_dtype = dt;
  if (u.kind == UnitKind::Attn) {
    st.a = act(int64_t(T) * 3 * h);  // qkv
    g.M = T, g.N = 3 * h, g.K = h;
    g.A = op(st.ln->p, h, false);
    g.B = op(weight(d, L + "attn.qkv.w"), h, false);
    g.epi.c = st.a->p, g.epi.c_dtype = dt, g.epi.ldc = 3 * h, g.epi.bias = master(d, L + "attn.qkv.b");
    gemm(d, g);
    if (use_flash()) {
      // Fused attention: ctx and the per-row log-sum-exp (the stash replaces P).
      st.b = f32(int64_t(m_.mbs) * H * S);
      st.c = act(int64_t(T) * h);
      timed_attention(d, false, [&] {
        launches_ += wpk::flash_attn_fwd(attn_shape(), st.a->p, st.c->p, static_cast<float*>(st.b->p), cs);
      });
    } else {
      // S = Q K^T / sqrt(d), per (head, sequence)
      wpk::GemmProblem sg;
      sg.in_dtype = dt;
      sg.M = S, sg.N = S, sg.K = dh, sg.nb1 = H, sg.nb2 = m_.mbs;
      sg.causal = m_.causal ? wpk::kCausalSkipUpper : wpk::kCausalNone;
      sg.A = op(st.a->p, 3 * h, false, dh, int64_t(S) * 3 * h);
      sg.B = op(at(st.a, h, es), 3 * h, false, dh, int64_t(S) * 3 * h);
      sg.epi.c = d.scores, sg.epi.c_dtype = wpk::kF32, sg.epi.ldc = S, sg.epi.c_b1 = int64_t(S) * S,
      sg.epi.c_b2 = int64_t(H) * S * S, sg.epi.alpha = 1.0f / std::sqrt(static_cast<float>(dh));
      gemm(d, sg);
      st.b = act(int64_t(m_.mbs) * H * S * S);  // P
      launches_ += wpk::softmax_fwd(dt, d.scores, st.b->p, m_.mbs * H * S, S, m_.causal, cs);
      if (check_ops_enabled()) check_softmax(dt, d.scores, st.b->p, m_.mbs * H * S, S, m_.causal, cs);
      // ctx = P V
      st.c = act(int64_t(T) * h);
      wpk::GemmProblem pv;
      pv.in_dtype = dt;
      pv.M = S, pv.N = dh, pv.K = S, pv.nb1 = H, pv.nb2 = m_.mbs;
      pv.causal = m_.causal ? wpk::kCausalKUpToRow : wpk::kCausalNone;
      pv.A = op(st.b->p, S, false, int64_t(S) * S, int64_t(H) * S * S);
      pv.B = op(at(st.a, 2 * h, es), 3 * h, true, dh, int64_t(S) * 3 * h);
      pv.epi.c = st.c->p, pv.epi.c_dtype = dt, pv.epi.ldc = h, pv.epi.c_b1 = dh, pv.epi.c_b2 = int64_t(S) * h;
      gemm(d, pv);
    }
    BufPtr out = act(int64_t(T) * h);
    wpk::GemmProblem pr;
    pr.in_dtype = dt;
    pr.M = T, pr.N = h, pr.K = h;
    pr.A = op(st.c->p, h, false);
    pr.B = op(weight(d, L + "attn.proj.w"), h, false);
    pr.epi.mode = wpk::kEpiResidual, pr.epi.c = out->p, pr.epi.c_dtype = dt, pr.epi.ldc = h,
    pr.epi.bias = master(d, L + "attn.proj.b"), pr.epi.resid = x->p;
    gemm(d, pr);
    return out;
  }
  if (u.kind == UnitKind::Mlp) {
    st.a = act(int64_t(T) * f);  // pre-activation u
    st.b = act(int64_t(T) * f);  // gelu(u)
    g.M = T, g.N = f, g.K = h;
    g.A = op(st.ln->p, h, false);
    g.B = op(weight(d, L + "mlp.fc1.w"), h, false);
    g.epi.mode = wpk::kEpiGelu, g.epi.c = st.b->p, g.epi.aux = st.a->p, g.epi.c_dtype = dt, g.epi.ldc = f,
    g.epi.bias = master(d, L + "mlp.fc1.b");
    gemm(d, g);
    BufPtr out = act(int64_t(T) * h);
    wpk::GemmProblem g2;
    g2.in_dtype = dt;
    g2.M = T, g2.N = h, g2.K = f;
    g2.A = op(st.b->p, f, false);
    g2.B = op(weight(d, L + "mlp.fc2.w"), f, false);
    g2.epi.mode = wpk::kEpiResidual, g2.epi.c = out->p, g2.epi.c_dtype = dt, g2.epi.ldc = h,
    g2.epi.bias = master(d, L + "mlp.fc2.b"), g2.epi.resid = x->p;
    gemm(d, g2);
    return out;
  }
  // Head: logits, fused cross-entropy (loss + dlogits in place).
  st.a = act(int64_t(T) * V);
  g.M = T, g.N = V, g.K = h;
  g.A = op(st.ln->p, h, false);
  g.B = op(weight(d, m_.tie ? "wte" : "lm_head.w"), h, false);
  g.epi.c = st.a->p, g.epi.c_dtype = dt, g.epi.ldc = V;
  gemm(d, g);
  const float scale = 1.0f / (static_cast<float>(T) * list_.config.microbatches);
  // logits read once, dlogits written in place, labels
  timed_hbm(d, "cross_entropy", 2.0 * es * T * double(V) + 4.0 * T, [&] {
    launches_ += wpk::xent_fwd_bwd(dt, st.a->p, d.labels + int64_t(mb) * T, d.loss, T, V, scale, scale, cs);
  });
  return nullptr;
}

BufPtr Runtime::unit_bwd(DeviceState& d, int ui, int mb, UnitStash& st, BufPtr dy) {
  const Unit& u = units_[ui];
  const int T = m_.tokens(), h = m_.hidden, f = m_.ffn, V = m_.vocab, S = m_.seq, H = m_.heads, dh = m_.head_dim();
  const int es = m_.act_bytes(), dt = m_.dtype;
  cudaStream_t cs = d.compute;
  Pool& pool = *d.pool;
  auto act = [&](int64_t n) { return pool.alloc(n * es, cs, 0); };
  auto drop = [&](BufPtr& b) {
    pool.release(b, cs);
    b.reset();
  };
  const std::string L = "h." + std::to_string(u.layer) + ".";
  const bool dy_bias_done = d.dy_bias_done;  // set by the unit above (same slice) for this dy
  d.dy_bias_done = false;

  if (u.kind == UnitKind::Embed) {
    // dy and tokens in; the T touched fp32 wte-gradient rows and the wpe
    // gradient read-modify-written
    timed_hbm(d, "embedding_bwd", double(es) * T * h + 4.0 * T + 8.0 * (double(T) * h + double(S) * h), [&] {
      launches_ += wpk::embed_bwd(dt, d.tokens + int64_t(mb) * T, dy->p, grad(d, "wte"), grad(d, "wpe"), T, S, h,
                                  cs);
    });
    drop(dy);
    return nullptr;
  }
  // dX = dY W  (B N-major: W[k][n] with k = out features)
  // LayerNorm-backward fused into the dgrad GEMM producing dLN (bf16, the
  // CTA-pair kernel's shapes): the epilogue accumulates dw, db and the two
  // row sums, leaving dx to an elementwise pass.  WP_LN_UNFUSED=1 keeps the
  // standalone kernel (A/B switch).
  static const bool ln_unfused = std::getenv("WP_LN_UNFUSED") != nullptr;
  const bool ln_fused = !ln_unfused && dt == wpk::kBF16 && T >= 256 && h > 128 && h % 8 == 0 &&
                        std::getenv("WP_GEMM_NO_PAIR") == nullptr && std::getenv("WP_GEMM_NO_TMA_EPI") == nullptr;
  // Attention's Delta = rowsum(dO * O) out of the projection data-gradient
  // GEMM that produces dO (its epilogue dots each 64-column slab of dO with
  // the stashed O); WP_DELTA_UNFUSED=1 keeps the standalone pass (A/B).
  static const bool delta_unfused = std::getenv("WP_DELTA_UNFUSED") != nullptr;
  const bool delta_fused = !delta_unfused && use_flash() && dt == wpk::kBF16 && T >= 256 && h > 128 && h % 64 == 0 &&
                           dh % 64 == 0 && std::getenv("WP_GEMM_NO_PAIR") == nullptr &&
                           std::getenv("WP_GEMM_NO_TMA_EPI") == nullptr;
  auto dgrad = [&](const void* dY, int ld_dy, int n_out, const void* W, int n_in, void* dX, int mode = wpk::kEpiStore,
                   const void* aux = nullptr, float* colsum = nullptr, const std::string& ln_name = std::string(),
                   bool delta = false) {
    wpk::GemmProblem g;
    g.in_dtype = dt;
    g.M = T, g.N = n_in, g.K = n_out;
    g.A = op(dY, ld_dy, false);
    g.B = op(W, n_in, true);
    g.epi.mode = mode, g.epi.c = dX, g.epi.c_dtype = dt, g.epi.ldc = n_in, g.epi.aux = const_cast<void*>(aux);
    g.epi.colsum = colsum;
    if (ln_fused && !ln_name.empty()) {
      ck(cudaMemsetAsync(d.ln_rows, 0, sizeof(float) * 2 * size_t(T), cs), "ln rows reset");
      g.epi.ln_x = st.x->p, g.epi.ln_mean = static_cast<float*>(st.mean->p);
      g.epi.ln_rstd = static_cast<float*>(st.rstd->p), g.epi.ln_w = master(d, ln_name + ".w");
      g.epi.ln_dw = grad(d, ln_name + ".w"), g.epi.colsum = grad(d, ln_name + ".b"), g.epi.ln_rows = d.ln_rows;
    }
    if (delta) {
      ck(cudaMemsetAsync(d.attn_delta, 0, sizeof(float) * size_t(T) * H, cs), "delta reset");
      g.epi.rd_x = st.c->p, g.epi.rd_out = d.attn_delta, g.epi.rd_group = dh, g.epi.rd_seq = S;
    }
    gemm(d, g);
  };
  // dW += dY^T X  (both operands MN-major over the token dimension)
  auto wgrad = [&](const void* dY, int n_out, const void* X, int n_in, float* dW) {
    wpk::GemmProblem g;
    g.in_dtype = dt;
    g.M = n_out, g.N = n_in, g.K = T;
    g.A = op(dY, n_out, true);
    g.B = op(X, n_in, true);
    g.epi.mode = wpk::kEpiAccum, g.epi.c = dW, g.epi.c_dtype = wpk::kF32, g.epi.ldc = n_in;
    gemm(d, g);
  };
  // The unit below this one in the same slice (run next, same device) takes
  // dx as its dy: with the fused LayerNorm its bias gradient -- the column
  // sums of that dy -- comes out of the dx pass (proj.b below an MLP's ln2,
  // fc2.b below an attention block's ln1 or the final LayerNorm).
  static const bool bias_unfused = std::getenv("WP_BIAS_UNFUSED") != nullptr;  // A/B switch
  auto below_bias = [&]() -> float* {
    if (!ln_fused || bias_unfused || ui - 1 < d.bwd_unit_lo) return nullptr;
    const Unit& v = units_[ui - 1];
    const std::string Lv = "h." + std::to_string(v.layer) + ".";
    if (v.kind == UnitKind::Attn) return grad(d, Lv + "attn.proj.b");
    if (v.kind == UnitKind::Mlp) return grad(d, Lv + "mlp.fc2.b");
    return nullptr;
  };
  auto ln_bwd = [&](const BufPtr& dln, const std::string& name, const BufPtr& dres) {
    BufPtr dx = act(int64_t(T) * h);
    if (ln_fused) {  // dw, db, row sums came with dLN from the dgrad GEMM
      float* dcol = below_bias();
      // dLN, x, (dres) in, dx out; mean, rstd, two row sums; w; bias-sum RMW
      const double bytes = double(es) * T * h * (dres ? 4.0 : 3.0) + 16.0 * T + 4.0 * h + (dcol ? 8.0 * h : 0.0);
      timed_hbm(d, "layernorm_bwd_dx", bytes, [&] {
        launches_ += wpk::layernorm_bwd_dx_rows(dt, dln->p, st.x->p, static_cast<float*>(st.mean->p),
                                                static_cast<float*>(st.rstd->p), master(d, name + ".w"), d.ln_rows,
                                                dres ? dres->p : nullptr, dx->p, T, h, cs, dcol);
      });
      d.dy_bias_done = dcol != nullptr;
      return dx;
    }
    LnBwdCheck chk;
    if (check_ops_enabled())
      chk.before(dt, dln->p, st.x->p, static_cast<float*>(st.mean->p), static_cast<float*>(st.rstd->p),
                 master(d, name + ".w"), dres ? dres->p : nullptr, grad(d, name + ".w"), grad(d, name + ".b"), T, h,
                 cs);
    timed_hbm(d, "layernorm_bwd", double(es) * T * h * (dres ? 4.0 : 3.0) + 8.0 * T + 20.0 * h, [&] {
      launches_ += wpk::layernorm_bwd(dt, dln->p, st.x->p, static_cast<float*>(st.mean->p),
                                      static_cast<float*>(st.rstd->p), master(d, name + ".w"),
                                      dres ? dres->p : nullptr, dx->p, grad(d, name + ".w"), grad(d, name + ".b"), T,
                                      h, cs);
    });
    if (check_ops_enabled()) chk.after(dx->p, grad(d, name + ".w"), grad(d, name + ".b"), cs);
    return dx;
  };

  if (u.kind == UnitKind::Head) {
    const std::string wn = m_.tie ? "wte" : "lm_head.w";
    BufPtr dln = act(int64_t(T) * h);
    dgrad(st.a->p, V, V, weight(d, wn), h, dln->p, wpk::kEpiStore, nullptr, nullptr, "lnf");
    wgrad(st.a->p, V, st.ln->p, h, grad(d, wn));
    BufPtr dx = ln_bwd(dln, "lnf", nullptr);
    drop(dln);
    for (BufPtr* b : {&st.x, &st.ln, &st.mean, &st.rstd, &st.a}) drop(*b);
    if (dy) drop(dy);
    return dx;
  }
  if (u.kind == UnitKind::Mlp) {
    BufPtr du = act(int64_t(T) * f);
    // dU = (dY W2) * gelu'(U); the fc1 bias gradient (column sums of dU) in the same epilogue
    dgrad(dy->p, h, h, weight(d, L + "mlp.fc2.w"), f, du->p, wpk::kEpiDGelu, st.a->p, grad(d, L + "mlp.fc1.b"));
    wgrad(dy->p, h, st.b->p, f, grad(d, L + "mlp.fc2.w"));
    if (!dy_bias_done)
      timed_hbm(d, "bias_colsum", double(es) * T * h + 8.0 * h,
                [&] { launches_ += wpk::colsum_accum(dt, dy->p, grad(d, L + "mlp.fc2.b"), T, h, h, cs); });
    wgrad(du->p, f, st.ln->p, h, grad(d, L + "mlp.fc1.w"));
    BufPtr dln = act(int64_t(T) * h);
    dgrad(du->p, f, f, weight(d, L + "mlp.fc1.w"), h, dln->p, wpk::kEpiStore, nullptr, nullptr, L + "ln2");
    BufPtr dx = ln_bwd(dln, L + "ln2", dy);
    drop(du);
    drop(dln);
    drop(dy);
    for (BufPtr* b : {&st.x, &st.ln, &st.mean, &st.rstd, &st.a, &st.b}) drop(*b);
    return dx;
  }
  // Attention block.
  BufPtr dctx = act(int64_t(T) * h);
  dgrad(dy->p, h, h, weight(d, L + "attn.proj.w"), h, dctx->p, wpk::kEpiStore, nullptr, nullptr, std::string(),
        delta_fused);
  wgrad(dy->p, h, st.c->p, h, grad(d, L + "attn.proj.w"));
  if (!dy_bias_done)
    timed_hbm(d, "bias_colsum", double(es) * T * h + 8.0 * h,
              [&] { launches_ += wpk::colsum_accum(dt, dy->p, grad(d, L + "attn.proj.b"), T, h, h, cs); });
  BufPtr dqkv;
  if (use_flash()) {
    dqkv = act(int64_t(T) * 3 * h);
    timed_attention(d, true, [&] {
      launches_ += wpk::flash_attn_bwd(attn_shape(), st.a->p, st.c->p, dctx->p, static_cast<float*>(st.b->p),
                                       d.attn_delta, d.dq_acc, dqkv->p, cs, grad(d, L + "attn.qkv.b"),
                                       delta_fused);
    });
  } else {
    // dP = dctx V^T  (fp32 scratch)
    {
      wpk::GemmProblem g;
      g.in_dtype = dt;
      g.M = S, g.N = S, g.K = dh, g.nb1 = H, g.nb2 = m_.mbs;
      g.causal = m_.causal ? wpk::kCausalSkipUpper : wpk::kCausalNone;
      g.A = op(dctx->p, h, false, dh, int64_t(S) * h);
      g.B = op(at(st.a, 2 * h, es), 3 * h, false, dh, int64_t(S) * 3 * h);
      g.epi.c = d.scores, g.epi.c_dtype = wpk::kF32, g.epi.ldc = S, g.epi.c_b1 = int64_t(S) * S,
      g.epi.c_b2 = int64_t(H) * S * S;
      gemm(d, g);
    }
    dqkv = act(int64_t(T) * 3 * h);
    // dV = P^T dctx
    {
      wpk::GemmProblem g;
      g.in_dtype = dt;
      g.M = S, g.N = dh, g.K = S, g.nb1 = H, g.nb2 = m_.mbs;
      g.causal = m_.causal ? wpk::kCausalKFromRow : wpk::kCausalNone;
      g.A = op(st.b->p, S, true, int64_t(S) * S, int64_t(H) * S * S);
      g.B = op(dctx->p, h, true, dh, int64_t(S) * h);
      g.epi.c = at(dqkv, 2 * h, es), g.epi.c_dtype = dt, g.epi.ldc = 3 * h, g.epi.c_b1 = dh,
      g.epi.c_b2 = int64_t(S) * 3 * h;
      gemm(d, g);
    }
    // dS = P * (dP - rowsum(dP * P)) / sqrt(d), in place over P
    launches_ += wpk::softmax_bwd(dt, d.scores, st.b->p, m_.mbs * H * S, S, 1.0f / std::sqrt(static_cast<float>(dh)),
                                  m_.causal, cs);
    // dQ = dS K
    {
      wpk::GemmProblem g;
      g.in_dtype = dt;
      g.M = S, g.N = dh, g.K = S, g.nb1 = H, g.nb2 = m_.mbs;
      g.causal = m_.causal ? wpk::kCausalKUpToRow : wpk::kCausalNone;
      g.A = op(st.b->p, S, false, int64_t(S) * S, int64_t(H) * S * S);
      g.B = op(at(st.a, h, es), 3 * h, true, dh, int64_t(S) * 3 * h);
      g.epi.c = dqkv->p, g.epi.c_dtype = dt, g.epi.ldc = 3 * h, g.epi.c_b1 = dh, g.epi.c_b2 = int64_t(S) * 3 * h;
      gemm(d, g);
    }
    // dK = dS^T Q
    {
      wpk::GemmProblem g;
      g.in_dtype = dt;
      g.M = S, g.N = dh, g.K = S, g.nb1 = H, g.nb2 = m_.mbs;
      g.causal = m_.causal ? wpk::kCausalKFromRow : wpk::kCausalNone;
      g.A = op(st.b->p, S, true, int64_t(S) * S, int64_t(H) * S * S);
      g.B = op(st.a->p, 3 * h, true, dh, int64_t(S) * 3 * h);
      g.epi.c = at(dqkv, h, es), g.epi.c_dtype = dt, g.epi.ldc = 3 * h, g.epi.c_b1 = dh,
      g.epi.c_b2 = int64_t(S) * 3 * h;
      gemm(d, g);
    }
  }
  wgrad(dqkv->p, 3 * h, st.ln->p, h, grad(d, L + "attn.qkv.w"));
  if (!use_flash())  // the fused attention backward sums the QKV bias gradient itself
    launches_ += wpk::colsum_accum(dt, dqkv->p, grad(d, L + "attn.qkv.b"), T, 3 * h, 3 * h, cs);
  BufPtr dln = act(int64_t(T) * h);
  dgrad(dqkv->p, 3 * h, 3 * h, weight(d, L + "attn.qkv.w"), h, dln->p, wpk::kEpiStore, nullptr, nullptr, L + "ln1");
  BufPtr dx = ln_bwd(dln, L + "ln1", dy);
  drop(dctx);
  drop(dqkv);
  drop(dln);
  drop(dy);
  for (BufPtr* b : {&st.x, &st.ln, &st.mean, &st.rstd, &st.a, &st.b, &st.c}) drop(*b);
  return dx;
}

// ---------------------------------------------------------- message plumbing
BufPtr Runtime::take_input(DeviceState& d, const MsgKey& k) {
  for (auto* box : {&d.handoff, &d.inbox}) {
    auto it = box->find(k);
    if (it != box->end()) {
      BufPtr b = it->second;
      box->erase(it);
      return b;
    }
  }
  throw wavepipe::SimulationError("runtime: input message (payload " + std::to_string(k.payload) + ", microbatch " +
                                  std::to_string(k.mb) + ", boundary " + std::to_string(k.low) + ") never arrived");
}

void Runtime::deliver(DeviceState& d, const MsgKey& k, BufPtr buf) {
  const int consumer = k.payload == kAct ? k.low + 1 : k.low;
  if (owner_device(k.mb, consumer) == d.pipe) {
    d.handoff[k] = buf;
    return;
  }
  d.outbox[k] = buf;
  cudaEvent_t e = next_event(d);
  ck(cudaEventRecord(e, d.compute), "record ready");
  d.outbox_ready[k] = e;
}

void Runtime::post_copy(DeviceState& dst, const MsgKey& k, Published msg) {
  DeviceState& src = *devs_[dev_of_pipeline_[msg.src]];
  const size_t bytes = msg.buf->bytes;
  BufPtr landing = dst.pool->alloc(bytes, src.copy, 1);
  cudaEvent_t post = dst.last_start ? dst.last_start : dst.step_begin;
  ck(cudaStreamWaitEvent(src.copy, post, 0), "wait post");
  ck(cudaStreamWaitEvent(src.copy, msg.ready, 0), "wait ready");
  if (src.cuda == dst.cuda) {
    ck(cudaMemcpyAsync(landing->p, msg.buf->p, bytes, cudaMemcpyDeviceToDevice, src.copy), "D2D copy");
  } else {
    ck(cudaMemcpyPeerAsync(landing->p, dst.cuda, msg.buf->p, src.cuda, bytes, src.copy), "peer copy");
  }
  cudaEvent_t arrive = next_event(src);
  ck(cudaEventRecord(arrive, src.copy), "record arrival");
  src.pool->release(msg.buf, src.copy);
  dst.pending.push_back(arrive);
  dst.inbox[k] = landing;
  if (tracing_) dst.comm_recs.push_back({msg.src, dst.pipe, post, arrive, &dst, &src});
}

// --------------------------------------------------------------- execution
void Runtime::forward(DeviceState& d, const Action& a) {
  const int b = a.microbatch, s = a.slice_index;
  BufPtr x = s == 0 ? nullptr : take_input(d, MsgKey{kAct, b, s - 1});
  SliceStash& st = d.stash[{b, s}];
  st.units.assign(bounds_[s + 1] - bounds_[s], UnitStash{});
  for (int u = bounds_[s]; u < bounds_[s + 1]; ++u) x = unit_fwd(d, u, b, x, st.units[u - bounds_[s]]);
  st.bytes = stash_bytes(st);
  d.live_stash += st.bytes;
  d.peak_stash = std::max(d.peak_stash, d.live_stash);
  int64_t& sb = d.slice_stash_bytes[s];
  sb = std::max(sb, st.bytes);
  if (s < list_.config.stages - 1) deliver(d, MsgKey{kAct, b, s}, x);
}

int64_t Runtime::stash_bytes(const SliceStash& st) {
  std::vector<const Buf*> seen;
  int64_t n = 0;
  for (const UnitStash& u : st.units)
    for (const BufPtr* b : {&u.x, &u.ln, &u.mean, &u.rstd, &u.a, &u.b, &u.c})
      if (*b && std::find(seen.begin(), seen.end(), b->get()) == seen.end()) {
        seen.push_back(b->get());
        n += static_cast<int64_t>((*b)->bytes);
      }
  return n;
}

void Runtime::stash_stats(int pipe, int64_t* peak_bytes, int64_t* slice_bytes, int nslices) const {
  if (pipe < 0 || pipe >= list_.config.devices || dev_of_pipeline_[pipe] < 0) {
    throw wavepipe::ConfigError("stash_stats: pipeline device is not local to this process");
  }
  const DeviceState& d = *devs_[dev_of_pipeline_[pipe]];
  *peak_bytes = d.peak_stash;
  for (int s = 0; s < nslices; ++s) {
    auto it = d.slice_stash_bytes.find(s);
    slice_bytes[s] = it == d.slice_stash_bytes.end() ? 0 : it->second;
  }
}

void Runtime::backward(DeviceState& d, const Action& a) {
  const int b = a.microbatch, s = a.slice_index;
  BufPtr dy = s == list_.config.stages - 1 ? nullptr : take_input(d, MsgKey{kGrad, b, s});
  auto it = d.stash.find({b, s});
  if (it == d.stash.end()) throw wavepipe::SimulationError("runtime: backward before forward");
  SliceStash st = std::move(it->second);
  d.stash.erase(it);
  const int64_t freed = st.bytes;
  d.bwd_unit_lo = bounds_[s];
  d.dy_bias_done = false;
  for (int u = bounds_[s + 1] - 1; u >= bounds_[s]; --u) dy = unit_bwd(d, u, b, st.units[u - bounds_[s]], dy);
  d.live_stash -= freed;
  d.dy_bias_done = false;
  if (s > 0) deliver(d, MsgKey{kGrad, b, s - 1}, dy);
}

void Runtime::optimizer(DeviceState& d) {
  if (grad_group_.size() > 1) dp_allreduce(d);
  if (!update_) return;
  wpk::OptimArgs o{m_.optimizer, m_.lr, m_.beta1, m_.beta2, m_.eps, m_.weight_decay, step_ + 1};
  // per parameter: master, grad (read, then zeroed), m, v read + written,
  // the bf16 shadow written
  const double per = (m_.optimizer == 1 ? 32.0 : 16.0) + (d.shadow ? 2.0 : 0.0);
  timed_hbm(d, "optimizer", per * double(d.nparam), [&] {
    launches_ += wpk::optimizer_step(o, d.master, d.grad, d.m, d.v, d.shadow, d.nparam, d.compute);
  });
}

// NVTX range per enqueued action ("dev 2 Forward mb 3 slice 5"), for
// timeline tools (nsys / ncu --nvtx); a no-op unless a tool is attached.
struct NvtxAction {
  bool on;
  NvtxAction(int dev, const Action& a) : on(nvtx_active()) {
    if (!on) return;
    char buf[96];
    std::snprintf(buf, sizeof buf, "dev %d %s mb %d slice %d", dev, wavepipe::action_kind_name(a.kind), a.microbatch,
                  a.slice_index);
    nvtxRangePushA(buf);
  }
  ~NvtxAction() {
    if (on) nvtxRangePop();
  }
  static bool nvtx_active() {
    static const bool active = std::getenv("NSYS_PROFILING_SESSION_ID") || std::getenv("NVTX_INJECTION64_PATH") ||
                               std::getenv("WP_NVTX");
    return active;
  }
};

bool Runtime::advance(DeviceState& d) {
  const auto& prog = list_.per_device[d.pipe];
  bool moved = false;
  DevGuard g(d.cuda);
  while (d.pc < prog.size()) {
    const Action& a = prog[d.pc];
    NvtxAction range(d.pipe, a);
    if (a.is_compute()) {
      for (cudaEvent_t e : d.pending) ck(cudaStreamWaitEvent(d.compute, e, 0), "wait arrival");
      d.pending.clear();
      if (!d.pending_ipc.empty()) ipc_land(d, a);
      d.last_start = next_event(d);
      ck(cudaEventRecord(d.last_start, d.compute), "record start");
      d.starts.push_back({d.pc, d.last_start});
      if (a.kind == ActionKind::Forward) forward(d, a);
      else backward(d, a);
      if (tracing_) {
        cudaEvent_t e = next_event(d);
        ck(cudaEventRecord(e, d.compute), "record end");
        d.recs.push_back({static_cast<int>(d.pc), a.kind, a.microbatch, a.slice_index, d.last_start, e});
      }
    } else if (a.kind == ActionKind::OptimizerStep) {
      optimizer(d);
    } else if (transport_ == WP_TRANSPORT_IPC) {
      if (a.kind == ActionKind::Receive) {
        ipc_post(d, message_key(a));
      } else {
        ipc_send(d, a);
        if (a.kind == ActionKind::BatchedExchange) {
          const auto [q, qi] = d.be_partner[d.pc];
          ipc_post(d, message_key(list_.per_device[q][qi]));
        }
      }
    } else {
      // In-process transport.
      auto publish = [&](const MsgKey& k) {
        auto it = d.outbox.find(k);
        if (it == d.outbox.end()) throw wavepipe::SimulationError("runtime: send before its producer");
        published_[k] = Published{d.pipe, it->second, d.outbox_ready[k]};
        d.outbox.erase(it);
        d.outbox_ready.erase(k);
      };
      if (a.kind == ActionKind::Send) {
        publish(message_key(a));
      } else if (a.kind == ActionKind::Receive) {
        auto it = published_.find(message_key(a));
        if (it == published_.end()) break;  // sender has not produced it yet
        Published msg = it->second;
        published_.erase(it);
        post_copy(d, message_key(a), msg);
      } else {  // BatchedExchange
        if (!d.published_at[d.pc]) {
          publish(message_key(a));
          d.published_at[d.pc] = 1;
        }
        const auto [q, qi] = d.be_partner[d.pc];
        const MsgKey kin = message_key(list_.per_device[q][qi]);
        auto it = published_.find(kin);
        if (it == published_.end()) break;  // counterpart not at the exchange yet
        Published msg = it->second;
        published_.erase(it);
        // An exchange has no prefetch anchor of its own: it moves as soon as
        // both sides reach it (ref src/simulate.cpp:134-155).
        cudaEvent_t saved = d.last_start;
        d.last_start = d.step_begin;
        post_copy(d, kin, msg);
        d.last_start = saved;
      }
    }
    ++d.pc;
    moved = true;
  }
  return moved;
}

void Runtime::enqueue_step() {
  for (bool moved = true; moved;) {
    moved = false;
    for (auto& d : devs_) moved = advance(*d) || moved;
  }
  for (auto& d : devs_) {
    if (d->pc < list_.per_device[d->pipe].size()) {
      throw wavepipe::SimulationError("runtime stalled: device " + std::to_string(d->pipe) + " blocked at " +
                                      wavepipe::describe_action(list_.per_device[d->pipe][d->pc]));
    }
  }
}

float Runtime::train_step(const int32_t* tokens, const int32_t* labels, bool on_device, cudaStream_t producer) {
  if (broken_) throw wavepipe::SimulationError("runtime: a previous step stalled; create a new runtime");
  if (transport_ == WP_TRANSPORT_IPC && !ipc_connected_) {
    throw wavepipe::ConfigError("IPC transport: call ipc_connect with every rank's handle before the first step");
  }
  epoch_ = static_cast<uint32_t>(step_ + 1);
  for (auto& kv : ipc_send_next_) kv.second = 0;
  const size_t n = size_t(list_.config.microbatches) * m_.tokens();
  if (on_device) {
    // Device inputs: order the copies below after the producer's writes (the
    // runtime's streams are non-blocking, so nothing else would).
    cudaPointerAttributes attr{};
    ck(cudaPointerGetAttributes(&attr, tokens), "token pointer attributes");
    if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged) {
      throw wavepipe::ConfigError("train_step: on_device set but tokens are not device memory");
    }
    DevGuard g(attr.device);
    if (!input_ready_ || input_ready_dev_ != attr.device) {
      if (input_ready_) {
        DevGuard g0(input_ready_dev_);
        cudaEventDestroy(input_ready_);
      }
      ck(cudaEventCreateWithFlags(&input_ready_, cudaEventDisableTiming), "event create");
      input_ready_dev_ = attr.device;
    }
    ck(cudaEventRecord(input_ready_, producer), "record input ready");
  }
  for (auto& d : devs_) {
    DevGuard g(d->cuda);
    if (on_device) ck(cudaStreamWaitEvent(d->compute, input_ready_, 0), "wait input producer");
    ck(cudaMemcpyAsync(d->tokens, tokens, n * sizeof(int32_t), on_device ? cudaMemcpyDefault : cudaMemcpyHostToDevice,
                       d->compute),
       "tokens H2D");
    ck(cudaMemcpyAsync(d->labels, labels, n * sizeof(int32_t), on_device ? cudaMemcpyDefault : cudaMemcpyHostToDevice,
                       d->compute),
       "labels H2D");
    ck(cudaMemsetAsync(d->loss, 0, sizeof(float), d->compute), "loss reset");
    if (!update_) ck(cudaMemsetAsync(d->grad, 0, d->nparam * sizeof(float), d->compute), "grad reset");
    d->pc = 0;
    d->ev_next = 0;
    d->pending.clear();
    d->pending_ipc.clear();
    d->last_start = nullptr;
    d->recs.clear();
    d->comm_recs.clear();
    d->gemm_recs.clear();
    d->starts.clear();
    d->published_at.assign(list_.per_device[d->pipe].size(), 0);
    ck(cudaEventRecord(d->step_begin, d->compute), "record step begin");
    if (tracing_) {
      if (!d->clock_host) {
        void* mem = nullptr;
        ck(cudaHostAlloc(&mem, sizeof(uint64_t), cudaHostAllocMapped), "cudaHostAlloc clock word");
        d->clock_host = static_cast<uint64_t*>(mem);
        ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d->clock_dev), mem, 0), "clock word device pointer");
      }
      launches_ += wpk::stamp_globaltimer(d->clock_dev, d->compute);  // right after step_begin
    }
    ck(cudaStreamWaitEvent(d->copy, d->step_begin, 0), "copy after begin");
  }
  enqueue_step();
  finish_step();
  float loss = 0.f;
  for (auto& d : devs_) {
    DevGuard g(d->cuda);
    float l = 0.f;
    ck(cudaMemcpy(&l, d->loss, sizeof(float), cudaMemcpyDeviceToHost), "loss D2H");
    loss += l;
    if (!d->stash.empty() || !d->handoff.empty() || !d->inbox.empty() || !d->outbox.empty() ||
        !d->pending_ipc.empty() || !ipc_ready_.empty()) {
      throw wavepipe::SimulationError("runtime: state left over at the end of the step");
    }
  }
  if (tracing_) collect_trace();
  for (auto& d : devs_) {
    DevGuard g(d->cuda);
    for (const auto& r : d->gemm_recs) {
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, r.s, r.e), "gemm time");
      if (r.hbm) {
        auto& st = hbm_stats_[r.shape];
        ++st.n;
        st.flops += r.flops;
        st.seconds += 1e-3 * ms;
        continue;
      }
      if (r.attention) {
        attn_seconds_ += 1e-3 * ms;
        attn_flops_ += r.flops;
        ++attn_launches_;
      } else {
        prof_seconds_ += 1e-3 * ms;
        prof_flops_ += r.flops;
        ++prof_launches_;
      }
      auto& st = prof_shapes_[r.shape];
      ++st.n;
      st.flops += r.flops;
      st.seconds += 1e-3 * ms;
    }
  }
  ++step_;
  return loss;
}

// Stall watchdog (ref src/simulate.cpp:160-165, SimulationError "simulation
// stalled"; the executor contract's stall row, SURVEY.md 8a').  Every local
// stream gets a completion event; the host polls them against the stall
// timeout instead of blocking in cudaStreamSynchronize, so a dead, slow or
// mismatched peer -- whose flags this rank's streams wait on -- surfaces as
// an error naming the blocked action instead of a hang.
void Runtime::finish_step() {
  std::vector<std::pair<int, cudaEvent_t>> done;  // (cuda device, event)
  for (auto& d : devs_) {
    DevGuard g(d->cuda);
    std::vector<cudaStream_t> streams{d->compute, d->copy};
    if (d->sig) streams.push_back(d->sig);
    for (auto& kv : d->tx) streams.push_back(kv.second);
    for (cudaStream_t s : streams) {
      cudaEvent_t e = next_event(*d);
      ck(cudaEventRecord(e, s), "record stream done");
      done.push_back({d->cuda, e});
    }
  }
  static const bool dbg = std::getenv("WP_DEBUG_WATCHDOG") != nullptr;  // debugging aid
  if (dbg) std::fprintf(stderr, "[wp] step %d enqueued; waiting on %zu streams\n", step_, done.size());
  const auto t0 = std::chrono::steady_clock::now();
  auto sleep_us = std::chrono::microseconds(0);
  for (size_t i = 0; i < done.size();) {
    DevGuard g(done[i].first);
    const cudaError_t q = cudaEventQuery(done[i].second);
    if (q == cudaSuccess) {
      ++i;
      continue;
    }
    if (q != cudaErrorNotReady) ck(q, "step");
    const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (waited > stall_timeout_s_) stalled();
    // Spin briefly, then back off to 1 ms polls (a step is >= milliseconds).
    if (waited > 1e-3) sleep_us = std::min(std::chrono::microseconds(1000), sleep_us + std::chrono::microseconds(20));
    if (sleep_us.count()) std::this_thread::sleep_for(sleep_us);
  }
}

void Runtime::stalled() {
  if (std::getenv("WP_DEBUG_WATCHDOG")) std::fprintf(stderr, "[wp] stall detected\n");
  std::string where;
  for (auto& d : devs_) {
    DevGuard g(d->cuda);
    const auto& prog = list_.per_device[d->pipe];
    std::string what;
    for (const auto& [pc, ev] : d->starts) {
      if (cudaEventQuery(ev) == cudaErrorNotReady) {
        what = "blocked at " + wavepipe::describe_action(prog[pc]) + " (position " + std::to_string(pc) +
               "), waiting for its input";
        break;
      }
    }
    if (what.empty() && d->pc < prog.size()) what = "blocked at " + wavepipe::describe_action(prog[d->pc]);
    if (what.empty()) {
      what = cudaStreamQuery(d->compute) == cudaErrorNotReady
                 ? "every compute started; blocked at the OptimizerStep (gradient all-reduce)"
                 : "every compute done; a send is waiting for its receiver's post";
    }
    where += (where.empty() ? "" : "; ") + std::string("device ") + std::to_string(d->pipe) + " " + what;
  }
  cudaGetLastError();
  broken_ = true;
  // Release this rank's device-side waits: every wait of the step is on a
  // flag of this rank's own arena (arrive / posted / all-reduce ready, done),
  // so raising all of them to the epoch lets the streams drain and the
  // runtime be freed.  The step's results are garbage; the runtime refuses
  // further steps.
  // Release this rank's device-side waits: every wait of the step is a
  // bounded wait kernel (wpk::wait_flag) that also polls the host abort word,
  // so one host store lets the streams drain and the runtime be freed.  The
  // step's results are garbage; the runtime refuses further steps.
  if (abort_host_) *abort_host_ = 1u;
  const auto t0 = std::chrono::steady_clock::now();
  while (!released_ && std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 10.0) {
    bool busy = false;
    for (auto& d : devs_) {
      DevGuard g(d->cuda);
      for (cudaStream_t q : {d->compute, d->copy, d->sig})
        if (q && cudaStreamQuery(q) == cudaErrorNotReady) busy = true;
      for (auto& kv : d->tx)
        if (cudaStreamQuery(kv.second) == cudaErrorNotReady) busy = true;
    }
    released_ = !busy;
    if (busy) std::this_thread::sleep_for(std::chrono::milliseconds(1));
  }
  cudaGetLastError();
  if (std::getenv("WP_DEBUG_WATCHDOG")) std::fprintf(stderr, "[wp] device waits released: %d\n", int(released_));
  throw wavepipe::SimulationError("runtime stalled (no progress for " + std::to_string(stall_timeout_s_) +
                                  " s): " + where);
}

void Runtime::collect_trace() {
  step_clock_ns_ = devs_.front()->clock_host ? static_cast<int64_t>(*devs_.front()->clock_host) : 0;
  trace_ = wavepipe::SimTrace{};
  trace_.intervals.resize(list_.config.devices);
  auto rel = [](DeviceState* d, cudaEvent_t e) {
    float ms = 0.f;
    DevGuard g(d->cuda);
    ck(cudaEventElapsedTime(&ms, d->step_begin, e), "event time");
    return 1e-3 * ms;
  };
  for (auto& d : devs_) {
    for (const auto& r : d->recs) {
      wavepipe::TraceInterval iv;
      iv.action_index = r.idx;
      iv.kind = r.kind;
      iv.microbatch = r.mb;
      iv.slice_index = r.slice;
      iv.direction = wavepipe::microbatch_direction(list_.config, r.mb);
      iv.start = rel(d.get(), r.s);
      iv.end = rel(d.get(), r.e);
      trace_.makespan = std::max(trace_.makespan, iv.end);
      trace_.intervals[d->pipe].push_back(iv);
    }
    for (const auto& c : d->comm_recs) {
      wavepipe::CommEvent ev{c.src, c.dst, rel(c.post_dev, c.post), rel(c.arrive_dev, c.arrive)};
      trace_.makespan = std::max(trace_.makespan, ev.arrival_time);
      trace_.comm_events.push_back(ev);
    }
  }
  std::sort(trace_.comm_events.begin(), trace_.comm_events.end(),
            [](const wavepipe::CommEvent& x, const wavepipe::CommEvent& y) {
              return std::tie(x.arrival_time, x.post_time, x.src_device, x.dst_device) <
                     std::tie(y.arrival_time, y.post_time, y.src_device, y.dst_device);
            });
}

void Runtime::memory(int64_t* pool_bytes, int64_t* landing_bytes) const {
  int64_t pool = 0;
  for (const auto& d : devs_) pool += static_cast<int64_t>(d->pool->reserved());
  *pool_bytes = pool;
  *landing_bytes = ipc_arena_ ? static_cast<int64_t>(ipc_arena_bytes_ - ipc_flag_bytes_) : 0;
}

std::string Runtime::gemm_report() const {
  std::vector<std::pair<double, std::string>> rows;
  for (const auto& [k, v] : prof_shapes_) {
    char line[256];
    std::snprintf(line, sizeof line, "%-36s n=%6lld  %9.3f ms  %7.1f TFLOP/s\n", k.c_str(),
                  static_cast<long long>(v.n), 1e3 * v.seconds, v.seconds > 0 ? v.flops / v.seconds / 1e12 : 0.0);
    rows.emplace_back(v.seconds, line);
  }
  std::sort(rows.rbegin(), rows.rend());
  std::string out;
  for (auto& r : rows) out += r.second;
  return out;
}

// ------------------------------------------------------------- parameters
const ParamDesc& Runtime::param_desc(int i, bool* owned) const {
  const auto& ref = param_index_.at(param_names_.at(i));
  if (owned) *owned = ref.device >= 0;
  return ref.desc;
}

void Runtime::get_param(const std::string& name, float* host, int64_t n, bool want_grad) {
  auto it = param_index_.find(name);
  if (it == param_index_.end()) throw wavepipe::ConfigError("unknown or non-local parameter: " + name);
  if (n != it->second.desc.numel) throw wavepipe::ConfigError("size mismatch for " + name);
  DeviceState& d = *devs_[it->second.device];
  DevGuard g(d.cuda);
  ck(cudaDeviceSynchronize(), "sync");
  const float* src = (want_grad ? d.grad : d.master) + d.params[it->second.slot].offset;
  ck(cudaMemcpy(host, src, n * sizeof(float), cudaMemcpyDeviceToHost), "param D2H");
}

void Runtime::set_param(const std::string& name, const float* host, int64_t n) {
  auto it = param_index_.find(name);
  if (it == param_index_.end()) throw wavepipe::ConfigError("unknown or non-local parameter: " + name);
  if (n != it->second.desc.numel) throw wavepipe::ConfigError("size mismatch for " + name);
  DeviceState& d = *devs_[it->second.device];
  DevGuard g(d.cuda);
  ck(cudaDeviceSynchronize(), "sync");
  const int64_t off = d.params[it->second.slot].offset;
  // Stream-ordered copy: a plain cudaMemcpy from pageable memory may return
  // before its DMA lands, and the compute stream (non-blocking) would not
  // order the shadow cast after it.
  ck(cudaMemcpyAsync(d.master + off, host, n * sizeof(float), cudaMemcpyHostToDevice, d.compute), "param H2D");
  if (d.shadow) {
    launches_ += wpk::cast_f32_to_bf16(d.master + off, static_cast<__nv_bfloat16*>(d.shadow) + off, n, d.compute);
  }
  ck(cudaStreamSynchronize(d.compute), "sync");
}

}  // namespace wprt
