// wavepipe::Runtime / wavepipe::train_step (include/wavepipe/runtime.hpp):
// the C++ drop-in next to the reference's simulate(), over wprt::Runtime.
#include "wavepipe/runtime.hpp"

#include <cstring>

#include "runtime/runtime.hpp"

namespace wavepipe {

namespace {

wp_model_desc to_desc(const ModelSpec& m) {
  wp_model_desc d{};
  d.layers = m.layers, d.hidden = m.hidden, d.heads = m.heads, d.ffn = m.ffn, d.seq = m.seq, d.vocab = m.vocab;
  d.micro_batch_size = m.micro_batch_size;
  d.causal = m.causal, d.tie_embeddings = m.tie_embeddings;
  d.dtype = m.bf16 ? 1 : 0;
  d.optimizer = m.adamw ? 1 : 0;
  d.lr = m.lr, d.beta1 = m.beta1, d.beta2 = m.beta2, d.eps = m.eps, d.weight_decay = m.weight_decay;
  d.seed = m.seed;
  return d;
}

// Cheap identity of a list: config and per-device action counts.
int64_t signature(const ActionList& l) {
  int64_t h = l.config.devices * 1000003LL + l.config.microbatches * 1009LL + l.config.waves * 31LL +
              static_cast<int>(l.config.scheme);
  for (const auto& dev : l.per_device) h = h * 131 + static_cast<int64_t>(dev.size());
  return h;
}

}  // namespace

Runtime::Runtime(const ModelSpec& model, const ActionList& list, Transport transport, std::vector<int> device_ids,
                 int rank)
    : impl_(std::make_unique<wprt::Runtime>(to_desc(model), list, static_cast<int>(transport),
                                            device_ids.empty() ? nullptr : device_ids.data(), rank)),
      list_signature_(signature(list)) {}

Runtime::~Runtime() = default;

std::vector<uint8_t> Runtime::ipc_handle() const {
  std::vector<uint8_t> h(WP_IPC_HANDLE_BYTES);
  impl_->ipc_handle(h.data());
  return h;
}

void Runtime::ipc_connect(const std::vector<uint8_t>& all_handles, int nranks) {
  if (all_handles.size() != size_t(nranks) * WP_IPC_HANDLE_BYTES) throw ConfigError("ipc_connect: handle size");
  impl_->ipc_connect(all_handles.data(), nranks);
}

void Runtime::set_update(bool on) { impl_->set_update(on); }

std::vector<float> Runtime::param(const std::string& name, bool grad) {
  for (int i = 0; i < impl_->param_count(); ++i) {
    bool owned = false;
    const auto& d = impl_->param_desc(i, &owned);
    if (d.name == name) {
      std::vector<float> out(d.numel);
      impl_->get_param(name, out.data(), d.numel, grad);
      return out;
    }
  }
  throw ConfigError("unknown or non-local parameter: " + name);
}

void Runtime::set_param(const std::string& name, const std::vector<float>& values) {
  impl_->set_param(name, values.data(), static_cast<int64_t>(values.size()));
}

SimTrace train_step(const ActionList& list, Runtime& rt, const Batch& batch) {
  if (signature(list) != rt.list_signature_) throw ScheduleError("train_step: list differs from the runtime's");
  rt.impl_->set_tracing(true);
  rt.last_loss_ = rt.impl_->train_step(batch.tokens, batch.labels, batch.on_device);
  rt.impl_->set_tracing(false);
  return rt.impl_->trace();
}

}  // namespace wavepipe
