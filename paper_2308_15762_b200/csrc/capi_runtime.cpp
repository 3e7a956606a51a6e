// C ABI of the GPU runtime (include/wavepipe.h, "GPU runtime" section).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include <memory>

#include "capi_internal.hpp"
#include "runtime/runtime.hpp"

struct wp_runtime {
  std::unique_ptr<wprt::Runtime> rt;
  wp_trace trace_view;
};

using wpc::fail;
using wpc::map_exception;

extern "C" {

int wp_runtime_create(const wp_model_desc* model, const wp_list* list, int transport, const int* device_ids,
                      int rank, wp_runtime** out) {
  try {
    if (!model || !list || !out) return fail(WP_ERR_CONFIG, "null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      return fail(WP_ERR_CUDA, "no CUDA device available: the runtime has no CPU fallback");
    }
    auto* r = new wp_runtime;
    try {
      r->rt = std::make_unique<wprt::Runtime>(*model, list->list, transport, device_ids, rank);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

void wp_runtime_free(wp_runtime* rt) { delete rt; }

int wp_runtime_ipc_handle(wp_runtime* rt, void* out) {
  try {
    if (!rt || !out) return fail(WP_ERR_CONFIG, "null argument");
    rt->rt->ipc_handle(out);
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_runtime_ipc_connect(wp_runtime* rt, const void* handles, int nranks) {
  try {
    if (!rt || !handles) return fail(WP_ERR_CONFIG, "null argument");
    rt->rt->ipc_connect(handles, nranks);
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_runtime_attn_stats(const wp_runtime* rt, int64_t* launches, double* flops, double* seconds) {
  if (!rt || !launches || !flops || !seconds) return fail(WP_ERR_CONFIG, "null argument");
  rt->rt->attn_stats(launches, flops, seconds);
  return WP_OK;
}

int wp_runtime_memory(const wp_runtime* rt, int64_t* pool_bytes, int64_t* landing_bytes) {
  if (!rt || !pool_bytes || !landing_bytes) return fail(WP_ERR_CONFIG, "null argument");
  rt->rt->memory(pool_bytes, landing_bytes);
  return WP_OK;
}

int wp_runtime_stash(const wp_runtime* rt, int device, int64_t* peak_bytes, int64_t* slice_bytes, int nslices) {
  try {
    if (!rt || !peak_bytes || (nslices > 0 && !slice_bytes)) return fail(WP_ERR_CONFIG, "null argument");
    rt->rt->stash_stats(device, peak_bytes, slice_bytes, nslices);
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_runtime_ipc_status(const wp_runtime* rt, int* ok, char* msg, int capacity) {
  if (!rt || !ok) return fail(WP_ERR_CONFIG, "null argument");
  *ok = rt->rt->ipc_ok() ? 1 : 0;
  if (msg && capacity > 0) {
    const std::string& e = rt->rt->ipc_error();
    const size_t n = std::min<size_t>(e.size(), size_t(capacity) - 1);
    std::memcpy(msg, e.data(), n);
    msg[n] = 0;
  }
  return WP_OK;
}

int wp_train_step_stream(wp_runtime* rt, const int32_t* tokens, const int32_t* labels, int on_device,
                         void* producer_stream, float* loss) {
  try {
    if (!rt || !tokens || !labels) return fail(WP_ERR_CONFIG, "null argument");
    const float l =
        rt->rt->train_step(tokens, labels, on_device != 0, static_cast<cudaStream_t>(producer_stream));
    if (loss) *loss = l;
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_train_step(wp_runtime* rt, const int32_t* tokens, const int32_t* labels, int on_device, float* loss) {
  return wp_train_step_stream(rt, tokens, labels, on_device, nullptr, loss);
}

int wp_runtime_set_stall_timeout(wp_runtime* rt, double seconds) {
  if (!rt) return fail(WP_ERR_CONFIG, "null argument");
  if (!(seconds > 0)) return fail(WP_ERR_CONFIG, "stall timeout must be positive");
  rt->rt->set_stall_timeout(seconds);
  return WP_OK;
}

int wp_runtime_hbm_count(const wp_runtime* rt, int* classes) {
  if (!rt || !classes) return fail(WP_ERR_CONFIG, "null argument");
  *classes = rt->rt->hbm_count();
  return WP_OK;
}

int wp_runtime_hbm_stat(const wp_runtime* rt, int index, const char** name, int64_t* launches, double* bytes,
                        double* seconds) {
  if (!rt || !name || !launches || !bytes || !seconds) return fail(WP_ERR_CONFIG, "null argument");
  if (index < 0 || index >= rt->rt->hbm_count()) return fail(WP_ERR_CONFIG, "hbm class index out of range");
  rt->rt->hbm_stat(index, name, launches, bytes, seconds);
  return WP_OK;
}

int wp_runtime_trace(wp_runtime* rt, const wp_trace** trace) {
  if (!rt || !trace) return fail(WP_ERR_CONFIG, "null argument");
  rt->trace_view.trace = rt->rt->trace();
  wpc::refresh(&rt->trace_view);
  *trace = &rt->trace_view;
  return WP_OK;
}

int wp_runtime_step_clock(const wp_runtime* rt, int64_t* ns) {
  if (!rt || !ns) return fail(WP_ERR_CONFIG, "null argument");
  *ns = rt->rt->step_clock_ns();
  return WP_OK;
}

int wp_runtime_set_tracing(wp_runtime* rt, int enabled) {
  if (!rt) return fail(WP_ERR_CONFIG, "null argument");
  rt->rt->set_tracing(enabled != 0);
  return WP_OK;
}

int wp_runtime_set_update(wp_runtime* rt, int enabled) {
  if (!rt) return fail(WP_ERR_CONFIG, "null argument");
  rt->rt->set_update(enabled != 0);
  return WP_OK;
}

int wp_param_count(const wp_runtime* rt, int* count) {
  if (!rt || !count) return fail(WP_ERR_CONFIG, "null argument");
  *count = rt->rt->param_count();
  return WP_OK;
}

int wp_param_info(const wp_runtime* rt, int index, const char** name, int64_t* numel, int* owned) {
  try {
    if (!rt) return fail(WP_ERR_CONFIG, "null argument");
    bool own = false;
    const auto& d = rt->rt->param_desc(index, &own);
    if (name) *name = d.name.c_str();
    if (numel) *numel = d.numel;
    if (owned) *owned = own ? 1 : 0;
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_get_param(wp_runtime* rt, const char* name, float* host_out, int64_t numel) {
  try {
    if (!rt || !name || !host_out) return fail(WP_ERR_CONFIG, "null argument");
    rt->rt->get_param(name, host_out, numel, false);
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_set_param(wp_runtime* rt, const char* name, const float* host_in, int64_t numel) {
  try {
    if (!rt || !name || !host_in) return fail(WP_ERR_CONFIG, "null argument");
    rt->rt->set_param(name, host_in, numel);
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_get_grad(wp_runtime* rt, const char* name, float* host_out, int64_t numel) {
  try {
    if (!rt || !name || !host_out) return fail(WP_ERR_CONFIG, "null argument");
    rt->rt->get_param(name, host_out, numel, true);
    return WP_OK;
  } catch (...) {
    return map_exception();
  }
}

int wp_runtime_set_profiling(wp_runtime* rt, int enabled) {
  if (!rt) return fail(WP_ERR_CONFIG, "null argument");
  rt->rt->set_profiling(enabled != 0);
  if (enabled) rt->rt->reset_gemm_stats();
  return WP_OK;
}

int wp_runtime_gemm_stats(const wp_runtime* rt, int64_t* launches, double* flops, double* seconds) {
  if (!rt || !launches || !flops || !seconds) return fail(WP_ERR_CONFIG, "null argument");
  rt->rt->gemm_stats(launches, flops, seconds);
  return WP_OK;
}

int wp_runtime_gemm_report(const wp_runtime* rt, char* buf, int capacity) {
  if (!rt || !buf || capacity <= 0) return fail(WP_ERR_CONFIG, "null argument");
  const std::string r = rt->rt->gemm_report();
  const size_t n = std::min(r.size(), static_cast<size_t>(capacity - 1));
  std::memcpy(buf, r.data(), n);
  buf[n] = 0;
  return WP_OK;
}

int wp_runtime_launch_count(const wp_runtime* rt, int64_t* launches) {
  if (!rt || !launches) return fail(WP_ERR_CONFIG, "null argument");
  *launches = rt->rt->launches();
  return WP_OK;
}

}  // extern "C"
