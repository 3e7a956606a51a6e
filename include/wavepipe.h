/* wavepipe-b200 C ABI.
 *
 * The reference (`wavepipe`, /root/reference/proj) is a C++20 library with no
 * C ABI; its API is C++ only (exceptions, std::vector).  This header is the
 * plain-C boundary a foreign caller (ctypes, cgo, JNI, N-API) binds: opaque
 * handles, caller-owned output buffers or borrowed pointers that stay valid
 * until the owning handle is freed, and `int` status codes with the
 * reference CLI's taxonomy (proj/tools/main.cpp:37-40) plus one for the GPU:
 *
 *   WP_OK=0  WP_ERR_SEMANTIC=1  WP_ERR_CONFIG=2  WP_ERR_IO=3  WP_ERR_CUDA=4
 *
 * No exception crosses this boundary; the message of the last failure on
 * the calling thread is available from wp_last_error().
 *
 * Each entry point names the reference interface it replaces (file:line under
 * /root/reference/proj).  INTEGRATION.md shows the ctypes / cgo stubs.
 */
#ifndef WAVEPIPE_H_
#define WAVEPIPE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { WP_OK = 0, WP_ERR_SEMANTIC = 1, WP_ERR_CONFIG = 2, WP_ERR_IO = 3, WP_ERR_CUDA = 4 };

/* Scheme values match wavepipe::Scheme (include/wavepipe/config.hpp:34). */
enum { WP_GPIPE = 0, WP_DAPPLE = 1, WP_CHIMERA = 2, WP_CHIMERA_WAVE = 3, WP_HANAYO = 4 };
/* ActionKind values match include/wavepipe/action.hpp:49-56. */
enum { WP_FORWARD = 0, WP_BACKWARD = 1, WP_SEND = 2, WP_RECEIVE = 3,
       WP_BATCHED_EXCHANGE = 4, WP_OPTIMIZER_STEP = 5 };

/* ScheduleConfig, include/wavepipe/config.hpp:52-59 (same field order). */
typedef struct wp_config {
  int scheme, devices, microbatches, waves, replicas, stages;
} wp_config;

/* CostModel, include/wavepipe/cost_model.hpp:27-30. */
typedef struct wp_cost {
  double t_forward, t_backward, t_comm;
} wp_cost;

/* Action, include/wavepipe/action.hpp:74-81: seven ints, -1 = absent. */
typedef struct wp_action {
  int kind, microbatch, local_module_rank, slice_index, peer, payload, batch_group;
} wp_action;

/* TraceInterval, include/wavepipe/simulate.hpp:37-45. */
typedef struct wp_interval {
  int action_index, kind, microbatch, slice_index, direction;
  double start, end;
} wp_interval;

/* CommEvent, include/wavepipe/simulate.hpp:49-54. */
typedef struct wp_comm_event {
  int src_device, dst_device;
  double post_time, arrival_time;
} wp_comm_event;

typedef struct wp_list wp_list;   /* ActionList (config + placement + streams) */
typedef struct wp_trace wp_trace; /* SimTrace (abstract units or seconds) */

const char* wp_last_error(void);
const char* wp_version(void);

/* make_config, src/config.cpp:47-81. */
int wp_make_config(int scheme, int devices, int microbatches, int waves, int replicas,
                   wp_config* out);

/* make_placement (src/placement.cpp:70-83) + generate_schedule
 * (src/schedule.cpp:475-499).  Bit-exact with the reference. */
int wp_generate_schedule(const wp_config* cfg, const wp_cost* cost, wp_list** out);

/* An ActionList from caller-provided streams over make_placement(cfg):
 * counts[d] actions for device d, concatenated in `actions`. */
int wp_list_from_actions(const wp_config* cfg, const int* counts, const wp_action* actions,
                         wp_list** out);

/* insert_comm, src/schedule.cpp:333-473 (input: compute-only list). */
int wp_insert_comm(const wp_list* compute_only, wp_list** out);

int wp_list_config(const wp_list* list, wp_config* out);
/* Borrowed pointer to device d's stream; valid until wp_list_free. */
int wp_list_device(const wp_list* list, int device, const wp_action** actions, int* count);
/* Slice indices held by device d in local_module_rank order (StagePlacement). */
int wp_list_placement(const wp_list* list, int device, int* slice_index, int capacity, int* count);
void wp_list_free(wp_list* list);

/* serialize_action_list / parse_action_list, src/serialize.cpp:236-307:
 * byte-identical JSON.  The returned string is owned by the library; free it
 * with wp_string_free. */
int wp_serialize(const wp_list* list, char** json);
int wp_parse(const char* json, wp_list** out);
void wp_string_free(char* s);

/* validate_all, src/validate.cpp:529-536.  *ok = 1 when every check passes;
 * diagnostics (text, one line per violation) are copied into `report`
 * (truncated to `capacity`) when non-null. */
int wp_validate(const wp_list* list, int* ok, char* report, int capacity);

/* simulate, src/simulate.cpp:57-178. */
int wp_simulate(const wp_list* list, const wp_cost* cost, wp_trace** out);
int wp_trace_makespan(const wp_trace* trace, double* makespan);
int wp_trace_devices(const wp_trace* trace, int* devices);
int wp_trace_intervals(const wp_trace* trace, int device, const wp_interval** iv, int* count);
int wp_trace_comm_events(const wp_trace* trace, const wp_comm_event** ev, int* count);
void wp_trace_free(wp_trace* trace);
/* A trace assembled by the caller -- e.g. the measured traces of the ranks
 * of a multi-process job gathered into one -- so bubble_ratio and
 * memory_profile apply unchanged: `counts[d]` intervals of device d,
 * concatenated device-major, plus `n_events` comm events.  The makespan is
 * the latest interval end or arrival (src/simulate.cpp:166-169). */
int wp_trace_build(int devices, const int* counts, const wp_interval* intervals, int n_events,
                   const wp_comm_event* events, wp_trace** out);

/* trace_to_gantt, src/gantt.cpp:91-95: "svg" or "csv" rendering of a trace
 * (simulated or measured); *out is a NUL-terminated string freed with
 * wp_string_free. */
int wp_trace_to_gantt(const wp_trace* trace, const char* format, char** out);

/* compare + compare_to_csv / compare_to_json, src/analytics.cpp:221-331:
 * n requests (scheme, waves) at a shared device budget and microbatch count,
 * rows in ascending makespan; format 0 = CSV, 1 = JSON (the reference's
 * bytes); *out freed with wp_string_free.  wp_compare_measured builds the
 * same rows from measured traces (one per request, of lists[i]). */
int wp_compare(const int* schemes, const int* waves, int n, int budget_devices, int microbatches,
               const wp_cost* base_cost, int format, char** out);
int wp_compare_measured(const int* schemes, const int* waves, int n, int budget_devices, int microbatches,
                        const wp_trace* const* traces, const wp_list* const* lists, double t_comm, int format,
                        char** out);

/* bubble_ratio, src/analytics.cpp:32-46. */
int wp_bubble_ratio(const wp_trace* trace, double* out);
/* memory_profile, src/analytics.cpp:48-91: per device (num, den) pairs,
 * 2*devices int64 each. */
int wp_memory_profile(const wp_trace* trace, const wp_list* list, int64_t* weight_units,
                      int64_t* peak_activation_units);
/* analytic_bubble_hanayo_d (src/analytics.cpp:143-157), the exact Rational
 * form (:124-141, costs as num/den pairs) and the simplified form (:159-164). */
int wp_analytic_bubble(int devices, int waves, double t_forward, double t_backward,
                       double t_comm, double* out);
int wp_analytic_bubble_exact(int devices, int waves, const int64_t t_forward[2],
                             const int64_t t_backward[2], const int64_t t_comm[2],
                             int64_t out[2]);
int wp_analytic_bubble_simplified(int devices, int waves, int64_t out[2]);

/* ------------------------------------------------------------------------
 * GPU runtime: executes an ActionList on B200s (the reference's simulate()
 * replaced by real sm_100a kernels and NVLink transfers).  See
 * include/wavepipe/runtime.hpp for the C++ form `wavepipe::train_step`.
 */

/* ModelSpec: a GPT/BERT-like decoder stack.  dtype: 0 = fp32 (parity mode,
 * SIMT kernels), 1 = bf16 (tcgen05 tensor cores, fp32 master weights). */
typedef struct wp_model_desc {
  int layers, hidden, heads, ffn, seq, vocab;
  int micro_batch_size; /* sequences per microbatch */
  int causal;           /* 1 GPT (causal LM), 0 BERT-like (bidirectional, MLM labels) */
  int tie_embeddings;   /* 1: LM head shares the token embedding */
  int dtype;
  int optimizer;        /* 0 SGD, 1 AdamW */
  float lr, beta1, beta2, eps, weight_decay;
  uint64_t seed;        /* parameter init seed */
} wp_model_desc;

typedef struct wp_runtime wp_runtime;

/* Transport between pipeline devices:
 *  WP_TRANSPORT_LOCAL: every device of the list lives in this process;
 *    device d runs on CUDA ordinal device_ids[d] (ids may repeat: several
 *    pipeline devices sharing one GPU, each with its own streams).
 *  WP_TRANSPORT_IPC: one process per GPU; messages are copy-engine pushes
 *    over NVLink into the receiver's CUDA-IPC-mapped landing slots,
 *    signalled by stream memory operations (no SMs spent on transfers).
 *    With list config replicas D > 1 (data parallelism, the reference's
 *    bookkeeping-only D) the job has P * D ranks: rank =
 *    replica * P + pipeline device, every replica runs the list on its own
 *    microbatches and OptimizerStep first all-reduces (averages) the
 *    gradients of each stage across the D replicas with one peer-memory
 *    kernel over NVLink.  After creation every rank exports
 *    wp_runtime_ipc_handle, the caller all-gathers the handles (rank order)
 *    and passes them to wp_runtime_ipc_connect before the first step.
 *  (Value 1 is retired: the round-1 NCCL transport posted a step's receives
 *  up front, beyond the reference's memory bound, and was removed.) */
enum { WP_TRANSPORT_LOCAL = 0, WP_TRANSPORT_IPC = 2 };

int wp_runtime_create(const wp_model_desc* model, const wp_list* list, int transport,
                      const int* device_ids, int rank, wp_runtime** out);
void wp_runtime_free(wp_runtime* rt);
/* IPC transport handshake.  `out` receives WP_IPC_HANDLE_BYTES bytes;
 * `handles` holds nranks (= P * D) of them, rank-major. */
#define WP_IPC_HANDLE_BYTES 128
int wp_runtime_ipc_handle(wp_runtime* rt, void* out);
int wp_runtime_ipc_connect(wp_runtime* rt, const void* handles, int nranks);
/* After connect: *ok = 1 if every mapped peer accepted a probe copy and a
 * stream-memory-op write (the step's operations); else 0 and the reason in
 * `msg` (the caller should stop: there is no other transport). */
int wp_runtime_ipc_status(const wp_runtime* rt, int* ok, char* msg, int capacity);

/* One synchronous training step (all microbatches, flush, optimizer).
 * tokens/labels: int32 [B * micro_batch_size * seq], microbatch-major, in HOST
 * or DEVICE memory (`on_device`).  *loss = mean loss over microbatches.
 * The measured trace (seconds, device clocks aligned) is available from
 * wp_runtime_trace until the next step.
 * Stream contract for device inputs: the runtime's streams wait for all work
 * enqueued so far on the legacy default stream of the inputs' device (the
 * stream PyTorch uses unless told otherwise); wp_train_step_stream names the
 * producer stream (a cudaStream_t) explicitly.  Host inputs are read before
 * the call returns.
 * Stall watchdog (ref src/simulate.cpp:160-165): if the step's device work
 * has not finished within the stall timeout (wp_runtime_set_stall_timeout,
 * default 300 s or $WP_STALL_TIMEOUT_S) -- a dead, slow or mismatched peer
 * rank -- the call returns WP_ERR_SEMANTIC naming the blocked action, after
 * releasing this rank's pending device waits; the runtime then refuses
 * further steps (free it). */
int wp_train_step(wp_runtime* rt, const int32_t* tokens, const int32_t* labels, int on_device,
                  float* loss);
int wp_train_step_stream(wp_runtime* rt, const int32_t* tokens, const int32_t* labels, int on_device,
                         void* producer_stream, float* loss);
int wp_runtime_set_stall_timeout(wp_runtime* rt, double seconds);
int wp_runtime_trace(wp_runtime* rt, const wp_trace** trace);
/* %globaltimer (ns) on the device when the last traced step began -- the
 * origin of that step's measured trace.  Ranks of a multi-process job shift
 * their traces by (their value - the smallest) before merging them
 * (wp_trace_build), so the merged trace is on one device clock. */
int wp_runtime_step_clock(const wp_runtime* rt, int64_t* ns);
/* Enables per-action CUDA events (measured trace); off = no event overhead. */
int wp_runtime_set_tracing(wp_runtime* rt, int enabled);
/* Skip the optimizer update (gradients stay accumulated); for parity tests. */
int wp_runtime_set_update(wp_runtime* rt, int enabled);

/* Parameter access by global name ("wte", "wpe", "h.<l>.ln1.w", ...), fp32.
 * Only the process owning the parameter can read it (IPC transport). */
int wp_param_count(const wp_runtime* rt, int* count);
int wp_param_info(const wp_runtime* rt, int index, const char** name, int64_t* numel, int* owned);
int wp_get_param(wp_runtime* rt, const char* name, float* host_out, int64_t numel);
int wp_set_param(wp_runtime* rt, const char* name, const float* host_in, int64_t numel);
int wp_get_grad(wp_runtime* rt, const char* name, float* host_out, int64_t numel);

/* Device memory held by this process's pipeline devices: the stash /
 * message pool (grows to its steady state in the first step) and the IPC
 * landing slots (bytes). */
int wp_runtime_memory(const wp_runtime* rt, int64_t* pool_bytes, int64_t* landing_bytes);
/* Activation stash of local pipeline device `device` (the memory
 * memory_profile counts, ref src/analytics.cpp:48-91): peak live bytes over
 * the steps run so far, and per slice (nslices entries, normally
 * config.stages) the bytes of one (microbatch, slice) entry -- the slice's
 * input message plus every tensor its units saved for backward; 0 for
 * slices on other devices. */
int wp_runtime_stash(const wp_runtime* rt, int device, int64_t* peak_bytes, int64_t* slice_bytes, int nslices);
/* Number of this library's kernels launched since the runtime was created. */
int wp_runtime_launch_count(const wp_runtime* rt, int64_t* launches);
/* GEMM profiling: CUDA events around every tcgen05/SIMT GEMM launch on its
 * own stream, accumulated over the steps run while enabled (enabling resets). */
int wp_runtime_set_profiling(wp_runtime* rt, int enabled);
int wp_runtime_gemm_stats(const wp_runtime* rt, int64_t* launches, double* flops, double* seconds);
/* The same for the fused attention launches (algorithmic FLOPs: forward
 * 4*mbs*heads*seq^2*d, halved when causal; backward 2.5x). */
int wp_runtime_attn_stats(const wp_runtime* rt, int64_t* launches, double* flops, double* seconds);
/* Text table of the profiled GEMMs by shape (launches, time, TFLOP/s). */
int wp_runtime_gemm_report(const wp_runtime* rt, char* buf, int capacity);
/* The HBM-bound kernels timed the same way, by kernel class ("layernorm_fwd",
 * "layernorm_bwd_dx", "cross_entropy", "embedding_fwd", "embedding_bwd",
 * "optimizer", ...): count of classes, then per class its launches,
 * algorithmic bytes (reads + writes of the tensors it must touch) and summed
 * kernel seconds.  `name` stays valid until profiling is re-enabled. */
int wp_runtime_hbm_count(const wp_runtime* rt, int* classes);
int wp_runtime_hbm_stat(const wp_runtime* rt, int index, const char** name, int64_t* launches, double* bytes,
                        double* seconds);

#ifdef __cplusplus
}
#endif

#endif /* WAVEPIPE_H_ */
