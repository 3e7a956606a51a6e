"""ctypes binding of the C ABI in include/wavepipe.h (libwavepipe.so).

The library is built in-tree by `make` (see __graft_entry__.build()).  There is
no Python fallback: if the shared library is missing, importing this module
raises.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwavepipe.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())")

lib = C.CDLL(LIB_PATH)

WP_OK, WP_ERR_SEMANTIC, WP_ERR_CONFIG, WP_ERR_IO, WP_ERR_CUDA = range(5)


class wp_config(C.Structure):
    _fields_ = [(n, C.c_int) for n in
                ("scheme", "devices", "microbatches", "waves", "replicas", "stages")]


class wp_cost(C.Structure):
    _fields_ = [("t_forward", C.c_double), ("t_backward", C.c_double),
                ("t_comm", C.c_double)]


class wp_action(C.Structure):
    _fields_ = [(n, C.c_int) for n in
                ("kind", "microbatch", "local_module_rank", "slice_index", "peer",
                 "payload", "batch_group")]


class wp_interval(C.Structure):
    _fields_ = [("action_index", C.c_int), ("kind", C.c_int), ("microbatch", C.c_int),
                ("slice_index", C.c_int), ("direction", C.c_int),
                ("start", C.c_double), ("end", C.c_double)]


class wp_comm_event(C.Structure):
    _fields_ = [("src_device", C.c_int), ("dst_device", C.c_int),
                ("post_time", C.c_double), ("arrival_time", C.c_double)]


class wp_model_desc(C.Structure):
    _fields_ = [(n, C.c_int) for n in
                ("layers", "hidden", "heads", "ffn", "seq", "vocab", "micro_batch_size",
                 "causal", "tie_embeddings", "dtype", "optimizer")] + \
               [(n, C.c_float) for n in ("lr", "beta1", "beta2", "eps", "weight_decay")] + \
               [("seed", C.c_uint64)]


P = C.c_void_p
PP = C.POINTER(C.c_void_p)
I = C.c_int
IP = C.POINTER(C.c_int)
D = C.c_double
DP = C.POINTER(C.c_double)
I64P = C.POINTER(C.c_int64)

_SIGS = {
    "wp_last_error": (C.c_char_p, []),
    "wp_version": (C.c_char_p, []),
    "wp_make_config": (I, [I, I, I, I, I, C.POINTER(wp_config)]),
    "wp_generate_schedule": (I, [C.POINTER(wp_config), C.POINTER(wp_cost), PP]),
    "wp_list_from_actions": (I, [C.POINTER(wp_config), IP, C.POINTER(wp_action), PP]),
    "wp_insert_comm": (I, [P, PP]),
    "wp_list_config": (I, [P, C.POINTER(wp_config)]),
    "wp_list_device": (I, [P, I, C.POINTER(C.POINTER(wp_action)), IP]),
    "wp_list_placement": (I, [P, I, IP, I, IP]),
    "wp_list_free": (None, [P]),
    "wp_serialize": (I, [P, C.POINTER(C.c_void_p)]),
    "wp_parse": (I, [C.c_char_p, PP]),
    "wp_string_free": (None, [C.c_void_p]),
    "wp_validate": (I, [P, IP, C.c_char_p, I]),
    "wp_simulate": (I, [P, C.POINTER(wp_cost), PP]),
    "wp_trace_makespan": (I, [P, DP]),
    "wp_trace_devices": (I, [P, IP]),
    "wp_trace_intervals": (I, [P, I, C.POINTER(C.POINTER(wp_interval)), IP]),
    "wp_trace_comm_events": (I, [P, C.POINTER(C.POINTER(wp_comm_event)), IP]),
    "wp_trace_free": (None, [P]),
    "wp_trace_build": (I, [I, IP, C.POINTER(wp_interval), I, C.POINTER(wp_comm_event), PP]),
    "wp_trace_to_gantt": (I, [P, C.c_char_p, C.POINTER(C.c_void_p)]),
    "wp_compare": (I, [IP, IP, I, I, I, C.POINTER(wp_cost), I, C.POINTER(C.c_void_p)]),
    "wp_compare_measured": (I, [IP, IP, I, I, I, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), D, I,
                                C.POINTER(C.c_void_p)]),
    "wp_bubble_ratio": (I, [P, DP]),
    "wp_memory_profile": (I, [P, P, I64P, I64P]),
    "wp_analytic_bubble": (I, [I, I, D, D, D, DP]),
    "wp_analytic_bubble_exact": (I, [I, I, I64P, I64P, I64P, I64P]),
    "wp_analytic_bubble_simplified": (I, [I, I, I64P]),
    "wp_runtime_create": (I, [C.POINTER(wp_model_desc), P, I, IP, I, PP]),
    "wp_runtime_free": (None, [P]),
    "wp_runtime_ipc_handle": (I, [P, C.c_void_p]),
    "wp_runtime_ipc_connect": (I, [P, C.c_void_p, I]),
    "wp_runtime_ipc_status": (I, [P, IP, C.c_char_p, I]),
    "wp_train_step": (I, [P, C.c_void_p, C.c_void_p, I, C.POINTER(C.c_float)]),
    "wp_train_step_stream": (I, [P, C.c_void_p, C.c_void_p, I, C.c_void_p, C.POINTER(C.c_float)]),
    "wp_runtime_set_stall_timeout": (I, [P, D]),
    "wp_runtime_trace": (I, [P, PP]),
    "wp_runtime_set_tracing": (I, [P, I]),
    "wp_runtime_step_clock": (I, [P, I64P]),
    "wp_runtime_set_update": (I, [P, I]),
    "wp_param_count": (I, [P, IP]),
    "wp_param_info": (I, [P, I, C.POINTER(C.c_char_p), I64P, IP]),
    "wp_get_param": (I, [P, C.c_char_p, C.POINTER(C.c_float), C.c_int64]),
    "wp_set_param": (I, [P, C.c_char_p, C.POINTER(C.c_float), C.c_int64]),
    "wp_get_grad": (I, [P, C.c_char_p, C.POINTER(C.c_float), C.c_int64]),
    "wp_runtime_launch_count": (I, [P, I64P]),
    "wp_runtime_memory": (I, [P, I64P, I64P]),
    "wp_runtime_stash": (I, [P, I, I64P, I64P, I]),
    "wp_runtime_set_profiling": (I, [P, I]),
    "wp_runtime_gemm_stats": (I, [P, I64P, DP, DP]),
    "wp_runtime_gemm_report": (I, [P, C.c_char_p, I]),
    "wp_runtime_attn_stats": (I, [P, I64P, DP, DP]),
    "wp_runtime_hbm_count": (I, [P, IP]),
    "wp_runtime_hbm_stat": (I, [P, I, C.POINTER(C.c_char_p), I64P, DP, DP]),
}

EXPORTED = tuple(_SIGS)

MISSING = []  # declared in wavepipe.h but not exported (tests assert it is empty)
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name, None)
    if _fn is None:
        MISSING.append(_name)
        continue
    _fn.restype = _res
    _fn.argtypes = _args


class WavepipeError(RuntimeError):
    """Raised on a non-zero status; `code` follows the reference CLI taxonomy."""

    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ConfigError(WavepipeError, ValueError):
    pass


class ScheduleError(WavepipeError):
    pass


class CudaError(WavepipeError):
    pass


def check(status):
    if status == WP_OK:
        return
    msg = lib.wp_last_error().decode()
    if status == WP_ERR_CONFIG:
        raise ConfigError(status, msg)
    if status == WP_ERR_CUDA:
        raise CudaError(status, msg)
    raise ScheduleError(status, msg)
