// C++ face of the GPU runtime: the reference's abstract-time executor
// `simulate(ActionList, CostModel) -> SimTrace` (proj/include/wavepipe/
// simulate.hpp:77, proj/src/simulate.cpp:57-178) gets a real counterpart,
//
//   SimTrace train_step(const ActionList& list, Runtime& rt, const Batch& batch);
//
// which executes one synchronous training step of `list` on B200s and returns
// the *measured* trace (seconds, same SimTrace shape), so bubble_ratio /
// compute_metrics / trace_to_gantt apply unchanged.  The same runtime is
// exposed as a C ABI in wavepipe.h (wp_runtime_*, wp_train_step).
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "wavepipe/core.hpp"

namespace wprt {
class Runtime;
}

namespace wavepipe {

// A GPT-like (causal LM) or BERT-like (bidirectional) pre-LN decoder stack.
struct ModelSpec {
  int layers = 4, hidden = 256, heads = 4, ffn = 1024, seq = 128, vocab = 1024;
  int micro_batch_size = 2;  // sequences per microbatch
  bool causal = true;
  bool tie_embeddings = true;
  bool bf16 = false;          // false: fp32 parity mode (SIMT); true: tcgen05 bf16, fp32 masters
  bool adamw = false;         // false: SGD
  float lr = 1e-3f, beta1 = 0.9f, beta2 = 0.95f, eps = 1e-8f, weight_decay = 0.f;
  uint64_t seed = 1234;
};

enum class Transport {
  Local = 0,  // every pipeline device of the list in this process
  Ipc = 2,    // one process per GPU, copy-engine pushes into CUDA-IPC landing slots
};

// One step's inputs: int32 [microbatches, micro_batch_size, seq], microbatch-major.
struct Batch {
  const int32_t* tokens = nullptr;
  const int32_t* labels = nullptr;
  bool on_device = false;  // host (pinned or pageable) or device memory
};

class Runtime {
 public:
  // device_ids: CUDA ordinal per pipeline device (Local) or this rank's GPU
  // (Ipc); rank: replica * P + pipeline device (Ipc).
  Runtime(const ModelSpec& model, const ActionList& list, Transport transport = Transport::Local,
          std::vector<int> device_ids = {}, int rank = 0);
  ~Runtime();
  Runtime(const Runtime&) = delete;
  Runtime& operator=(const Runtime&) = delete;

  // IPC handshake (Transport::Ipc): export, all-gather out of band, connect.
  std::vector<uint8_t> ipc_handle() const;
  void ipc_connect(const std::vector<uint8_t>& all_handles, int nranks);

  float last_loss() const { return last_loss_; }
  void set_update(bool on);  // false: keep gradients, skip the optimizer (parity tests)
  std::vector<float> param(const std::string& name, bool grad = false);
  void set_param(const std::string& name, const std::vector<float>& values);
  wprt::Runtime& impl() { return *impl_; }

 private:
  friend SimTrace train_step(const ActionList& list, Runtime& rt, const Batch& batch);
  std::unique_ptr<wprt::Runtime> impl_;
  int64_t list_signature_ = 0;
  float last_loss_ = 0.f;
};

// One synchronous training step (every microbatch's forward and backward,
// the flush, the optimizer) of `list` -- the list the runtime was built
// with -- and its measured trace in seconds.  Throws ScheduleError on a list
// mismatch or a stalled program, std::runtime_error on CUDA errors.
SimTrace train_step(const ActionList& list, Runtime& rt, const Batch& batch);

}  // namespace wavepipe
