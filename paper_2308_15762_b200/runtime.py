"""GPU train-step runtime: executes a wavepipe ActionList on B200s.

Python face of `wp_runtime_*` / `wp_train_step` in include/wavepipe.h.  The
C++ runtime drives CUDA streams/events and the sm_100a kernels; this module
only marshals arguments.  There is no CPU fallback: creating a Runtime
without a CUDA device raises CudaError.
"""
import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._native import check, lib, wp_model_desc
from .schedule import ActionList, SimTrace

TRANSPORT_LOCAL = 0
TRANSPORT_IPC = 2
IPC_HANDLE_BYTES = 128


@dataclass
class ModelDesc:
    """ModelSpec of the stage compute (GPT-like causal LM or BERT-like)."""
    layers: int = 4
    hidden: int = 256
    heads: int = 4
    ffn: int = 1024
    seq: int = 128
    vocab: int = 1024
    micro_batch_size: int = 2
    causal: bool = True
    tie_embeddings: bool = True
    dtype: str = "fp32"          # "fp32" (parity mode) or "bf16"
    optimizer: str = "sgd"       # "sgd" or "adamw"
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.0
    seed: int = 1234

    def _c(self):
        return wp_model_desc(self.layers, self.hidden, self.heads, self.ffn, self.seq, self.vocab,
                             self.micro_batch_size, int(self.causal), int(self.tie_embeddings),
                             0 if self.dtype == "fp32" else 1, 0 if self.optimizer == "sgd" else 1,
                             self.lr, self.beta1, self.beta2, self.eps, self.weight_decay, self.seed)

    @property
    def tokens_per_microbatch(self):
        return self.micro_batch_size * self.seq

    def flops_per_sample(self):
        """3 x forward FLOPs: L*(2*(4h^2+2hf) + a*s*h) + 2hV per token."""
        a = 2 if self.causal else 4
        h, f, s = self.hidden, self.ffn, self.seq
        per_token = self.layers * (2 * (4 * h * h + 2 * h * f) + a * s * h) + 2 * h * self.vocab
        return 3.0 * s * per_token


def _all_gather_bytes(blob: bytes):
    """Default IPC handshake: all-gather over the initialised torch.distributed
    group (rank order)."""
    import torch.distributed as dist
    if not dist.is_initialized():
        raise RuntimeError("TRANSPORT_IPC needs torch.distributed initialised or an `exchange` callable")
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, blob)
    return out


class Runtime:
    """wp_runtime_create / wp_train_step.  transport:
    TRANSPORT_LOCAL  all pipeline devices in this process (device_ids[d] per device);
    TRANSPORT_IPC    one process per GPU, copy-engine pushes into CUDA-IPC-mapped
                     landing slots; with schedule.config.replicas = D > 1 the job
                     has P*D ranks (rank = replica*P + pipeline device) and the
                     optimizer step all-reduces gradients across replicas over
                     peer memory; `exchange(bytes) -> [bytes]*(P*D)` all-gathers
                     the handles (default: torch.distributed)."""

    def __init__(self, model: ModelDesc, schedule: ActionList, transport=TRANSPORT_LOCAL, device_ids=None,
                 rank=0, exchange=None, stall_timeout=None):
        self.model = model
        self.schedule = schedule
        P = schedule.config.devices
        n_ids = P if transport == TRANSPORT_LOCAL else 1
        ids = list(device_ids) if device_ids is not None else [0] * n_ids
        self._ids = (C.c_int * len(ids))(*ids)
        self._desc = model._c()
        h = C.c_void_p()
        check(lib.wp_runtime_create(C.byref(self._desc), schedule.handle, transport, self._ids, rank, C.byref(h)))
        self._h = h
        if stall_timeout is not None:
            self.set_stall_timeout(stall_timeout)
        if transport == TRANSPORT_IPC:
            mine = C.create_string_buffer(IPC_HANDLE_BYTES)
            check(lib.wp_runtime_ipc_handle(self._h, mine))
            blobs = (exchange or _all_gather_bytes)(mine.raw)
            world = P * max(1, schedule.config.replicas)
            if len(blobs) != world or any(len(b) != IPC_HANDLE_BYTES for b in blobs):
                raise ValueError(f"exchange must return one {IPC_HANDLE_BYTES}-byte handle per rank")
            allh = C.create_string_buffer(b"".join(blobs), world * IPC_HANDLE_BYTES)
            check(lib.wp_runtime_ipc_connect(self._h, allh, world))

    def set_stall_timeout(self, seconds):
        """Watchdog: a step whose device work makes no progress for `seconds`
        (a dead or mismatched peer) raises ScheduleError [1] naming the blocked
        action; the runtime is unusable afterwards."""
        check(lib.wp_runtime_set_stall_timeout(self._h, float(seconds)))

    def ipc_status(self):
        """(ok, message) of the IPC transport's set-up probe of its peers."""
        ok = C.c_int()
        msg = C.create_string_buffer(512)
        check(lib.wp_runtime_ipc_status(self._h, C.byref(ok), msg, len(msg)))
        return bool(ok.value), msg.value.decode()

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.wp_runtime_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    # --------------------------------------------------------------- steps
    def train_step(self, tokens, labels):
        """One synchronous step over all microbatches.  tokens/labels: int32
        [B, micro_batch_size, seq] as numpy arrays (host) or CUDA tensors
        (device; the step waits for torch's current stream, which produced
        them).  Returns the mean loss over microbatches."""
        on_dev = 0
        stream = None
        if hasattr(tokens, "is_cuda"):
            on_dev = int(tokens.is_cuda)
            if on_dev:
                import torch
                stream = torch.cuda.current_stream(tokens.device).cuda_stream
            tp, lp = tokens.data_ptr(), labels.data_ptr()
        else:
            tokens = np.ascontiguousarray(tokens, dtype=np.int32)
            labels = np.ascontiguousarray(labels, dtype=np.int32)
            tp, lp = tokens.ctypes.data, labels.ctypes.data
        loss = C.c_float()
        check(lib.wp_train_step_stream(self._h, C.c_void_p(tp), C.c_void_p(lp), on_dev, C.c_void_p(stream),
                                       C.byref(loss)))
        return loss.value

    def set_tracing(self, on=True):
        check(lib.wp_runtime_set_tracing(self._h, int(on)))

    def set_update(self, on=True):
        check(lib.wp_runtime_set_update(self._h, int(on)))

    def trace(self) -> SimTrace:
        """Measured trace of the last traced step (seconds)."""
        p = C.c_void_p()
        check(lib.wp_runtime_trace(self._h, C.byref(p)))
        return SimTrace(p, owned=False)

    def step_clock_ns(self):
        """%globaltimer (ns) when the last traced step began (its trace's origin)."""
        n = C.c_int64()
        check(lib.wp_runtime_step_clock(self._h, C.byref(n)))
        return n.value

    def launch_count(self):
        n = C.c_int64()
        check(lib.wp_runtime_launch_count(self._h, C.byref(n)))
        return n.value

    def memory(self):
        """(pool_bytes, landing_bytes): stash/message pool and IPC landing slots."""
        a, b = C.c_int64(), C.c_int64()
        check(lib.wp_runtime_memory(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def stash(self, device):
        """(peak live stash bytes, [bytes of one (microbatch, slice) entry per
        slice]) of local pipeline device `device`."""
        S = self.schedule.config.stages
        peak = C.c_int64()
        per = (C.c_int64 * S)()
        check(lib.wp_runtime_stash(self._h, device, C.byref(peak), per, S))
        return peak.value, list(per)

    def set_profiling(self, on=True):
        check(lib.wp_runtime_set_profiling(self._h, int(on)))

    def gemm_stats(self):
        """(launches, executed FLOPs, summed kernel seconds) of the GEMMs run
        while profiling was enabled."""
        n, fl, sec = C.c_int64(), C.c_double(), C.c_double()
        check(lib.wp_runtime_gemm_stats(self._h, C.byref(n), C.byref(fl), C.byref(sec)))
        return n.value, fl.value, sec.value

    def attn_stats(self):
        """(launches, algorithmic FLOPs, summed kernel seconds) of the fused
        attention launches run while profiling was enabled."""
        n, fl, sec = C.c_int64(), C.c_double(), C.c_double()
        check(lib.wp_runtime_attn_stats(self._h, C.byref(n), C.byref(fl), C.byref(sec)))
        return n.value, fl.value, sec.value

    def hbm_stats(self):
        """{kernel class: (launches, algorithmic bytes, summed seconds)} of the
        HBM-bound kernels run while profiling was enabled."""
        n = C.c_int()
        check(lib.wp_runtime_hbm_count(self._h, C.byref(n)))
        out = {}
        for i in range(n.value):
            name, k, b, sec = C.c_char_p(), C.c_int64(), C.c_double(), C.c_double()
            check(lib.wp_runtime_hbm_stat(self._h, i, C.byref(name), C.byref(k), C.byref(b), C.byref(sec)))
            out[name.value.decode()] = (k.value, b.value, sec.value)
        return out

    def gemm_report(self):
        buf = C.create_string_buffer(1 << 16)
        check(lib.wp_runtime_gemm_report(self._h, buf, len(buf)))
        return buf.value.decode()

    # ----------------------------------------------------------- parameters
    def param_names(self):
        n = C.c_int()
        check(lib.wp_param_count(self._h, C.byref(n)))
        out = []
        for i in range(n.value):
            name = C.c_char_p()
            numel = C.c_int64()
            owned = C.c_int()
            check(lib.wp_param_info(self._h, i, C.byref(name), C.byref(numel), C.byref(owned)))
            out.append((name.value.decode(), numel.value))
        return out

    def get_param(self, name, numel):
        buf = np.empty(numel, dtype=np.float32)
        check(lib.wp_get_param(self._h, name.encode(), buf.ctypes.data_as(C.POINTER(C.c_float)), numel))
        return buf

    def get_grad(self, name, numel):
        buf = np.empty(numel, dtype=np.float32)
        check(lib.wp_get_grad(self._h, name.encode(), buf.ctypes.data_as(C.POINTER(C.c_float)), numel))
        return buf

    def set_param(self, name, values):
        arr = np.ascontiguousarray(values, dtype=np.float32).ravel()
        check(lib.wp_set_param(self._h, name.encode(), arr.ctypes.data_as(C.POINTER(C.c_float)), arr.size))
