"""Python mirror of the reference's schedule API (namespace `wavepipe`).

Same names, argument meaning and error behaviour as the C++ headers under
/root/reference/proj/include/wavepipe/ (config.hpp, action.hpp,
cost_model.hpp, placement.hpp, schedule.hpp, simulate.hpp, analytics.hpp,
serialize.hpp, validate.hpp); every call goes through the C ABI of
libwavepipe.so (include/wavepipe.h).  Errors raise ConfigError (bad config /
parse, the reference's ConfigError/ParseError) or ScheduleError (semantic:
ScheduleError/SimulationError).
"""
import ctypes as C
import enum
from dataclasses import dataclass, field
from fractions import Fraction
from typing import List, NamedTuple

from ._native import (ConfigError, ScheduleError, check, lib, wp_action, wp_comm_event,
                      wp_config, wp_cost, wp_interval)

__all__ = [
    "compare", "compare_measured",
    "Scheme", "ActionKind", "Payload", "Direction", "ScheduleConfig", "CostModel", "Action",
    "ActionList", "TraceInterval", "CommEvent", "SimTrace", "build_trace", "trace_to_gantt", "make_config", "generate_schedule",
    "insert_comm", "simulate", "bubble_ratio", "memory_profile", "activation_variance",
    "analytic_bubble_hanayo", "analytic_bubble_hanayo_d", "analytic_bubble_simplified",
    "serialize_action_list", "parse_action_list", "validate_all", "ConfigError", "ScheduleError",
]


class Scheme(enum.IntEnum):
    GPipe = 0
    Dapple = 1
    Chimera = 2
    ChimeraWave = 3
    Hanayo = 4


class ActionKind(enum.IntEnum):
    Forward = 0
    Backward = 1
    Send = 2
    Receive = 3
    BatchedExchange = 4
    OptimizerStep = 5


class Payload(enum.IntEnum):
    Activation = 0
    Gradient = 1


class Direction(enum.IntEnum):
    Down = 0
    Up = 1


@dataclass(frozen=True)
class ScheduleConfig:
    scheme: Scheme = Scheme.GPipe
    devices: int = 1
    microbatches: int = 1
    waves: int = 1
    replicas: int = 1
    stages: int = 1

    def _c(self):
        return wp_config(int(self.scheme), self.devices, self.microbatches, self.waves, self.replicas,
                         self.stages)


@dataclass(frozen=True)
class CostModel:
    t_forward: float = 1.0
    t_backward: float = 2.0
    t_comm: float = 0.0

    def _c(self):
        return wp_cost(self.t_forward, self.t_backward, self.t_comm)

    def slice_forward(self, cfg):
        wave = cfg.scheme in (Scheme.Hanayo, Scheme.ChimeraWave)
        return self.t_forward / (2.0 * cfg.waves) if wave else self.t_forward

    def slice_backward(self, cfg):
        wave = cfg.scheme in (Scheme.Hanayo, Scheme.ChimeraWave)
        return self.t_backward / (2.0 * cfg.waves) if wave else self.t_backward

    def rescaled(self, budget_devices, config_devices):
        """ref include/wavepipe/cost_model.hpp:42-48: compute costs scaled by
        budget/config devices (one chimera-wave group of a budget)."""
        k = budget_devices / config_devices
        return CostModel(self.t_forward * k, self.t_backward * k, self.t_comm)


class Action(NamedTuple):
    kind: ActionKind
    microbatch: int = -1
    local_module_rank: int = -1
    slice_index: int = -1
    peer: int = -1
    payload: int = -1
    batch_group: int = -1

    def is_compute(self):
        return self.kind in (ActionKind.Forward, ActionKind.Backward)

    def is_comm(self):
        return self.kind in (ActionKind.Send, ActionKind.Receive, ActionKind.BatchedExchange)


class TraceInterval(NamedTuple):
    action_index: int
    kind: ActionKind
    microbatch: int
    slice_index: int
    direction: Direction
    start: float
    end: float


class CommEvent(NamedTuple):
    src_device: int
    dst_device: int
    post_time: float
    arrival_time: float


def make_config(scheme, devices, microbatches, waves=1, replicas=1):
    """make_config (ref src/config.cpp:47-81); raises ConfigError."""
    out = wp_config()
    check(lib.wp_make_config(int(scheme), devices, microbatches, waves, replicas, C.byref(out)))
    return ScheduleConfig(Scheme(out.scheme), out.devices, out.microbatches, out.waves, out.replicas,
                          out.stages)


class ActionList:
    """Owning wrapper of a wp_list handle (config + placement + per-device streams)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        cfg = wp_config()
        check(lib.wp_list_config(self._h, C.byref(cfg)))
        self.config = ScheduleConfig(Scheme(cfg.scheme), cfg.devices, cfg.microbatches, cfg.waves,
                                     cfg.replicas, cfg.stages)
        self._per_device = None
        self._placement = None

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.wp_list_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def per_device(self) -> List[List[Action]]:
        if self._per_device is None:
            out = []
            for d in range(self.config.devices):
                ptr = C.POINTER(wp_action)()
                n = C.c_int()
                check(lib.wp_list_device(self._h, d, C.byref(ptr), C.byref(n)))
                out.append([Action(ActionKind(a.kind), a.microbatch, a.local_module_rank, a.slice_index,
                                   a.peer, a.payload, a.batch_group) for a in ptr[:n.value]])
            self._per_device = out
        return self._per_device

    @property
    def placement(self) -> List[List[int]]:
        """Slice indices per device in local_module_rank order."""
        if self._placement is None:
            out = []
            for d in range(self.config.devices):
                n = C.c_int()
                check(lib.wp_list_placement(self._h, d, None, 0, C.byref(n)))
                buf = (C.c_int * max(1, n.value))()
                check(lib.wp_list_placement(self._h, d, buf, n.value, C.byref(n)))
                out.append(list(buf[:n.value]))
            self._placement = out
        return self._placement

    def compact(self):
        """Canonical text of the streams (one line per device); hashing key of
        the golden grid."""
        return "\n".join(";".join(",".join(str(int(x)) for x in a) for a in dev) for dev in self.per_device)

    @classmethod
    def from_actions(cls, cfg: ScheduleConfig, per_device):
        counts = (C.c_int * cfg.devices)(*[len(s) for s in per_device])
        flat = [a for s in per_device for a in s]
        arr = (wp_action * max(1, len(flat)))(*[wp_action(int(a[0]), *[int(x) for x in a[1:]]) for a in flat])
        h = C.c_void_p()
        c = cfg._c()
        check(lib.wp_list_from_actions(C.byref(c), counts, arr, C.byref(h)))
        return cls(h)


def generate_schedule(cfg: ScheduleConfig, cost: CostModel = None) -> ActionList:
    """make_placement + generate_schedule (ref src/schedule.cpp:475-499)."""
    cost = cost or CostModel()
    h = C.c_void_p()
    c, k = cfg._c(), cost._c()
    check(lib.wp_generate_schedule(C.byref(c), C.byref(k), C.byref(h)))
    return ActionList(h)


def insert_comm(compute_only: ActionList) -> ActionList:
    h = C.c_void_p()
    check(lib.wp_insert_comm(compute_only.handle, C.byref(h)))
    return ActionList(h)


class SimTrace:
    """SimTrace (ref include/wavepipe/simulate.hpp:56-60); abstract units from
    simulate(), seconds from the GPU runtime."""

    def __init__(self, handle, owned=True):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        self._owned = owned
        m = C.c_double()
        check(lib.wp_trace_makespan(self._h, C.byref(m)))
        self.makespan = m.value
        n = C.c_int()
        check(lib.wp_trace_devices(self._h, C.byref(n)))
        self.intervals = []
        for d in range(n.value):
            ptr = C.POINTER(wp_interval)()
            cnt = C.c_int()
            check(lib.wp_trace_intervals(self._h, d, C.byref(ptr), C.byref(cnt)))
            self.intervals.append([TraceInterval(i.action_index, ActionKind(i.kind), i.microbatch,
                                                 i.slice_index, Direction(i.direction), i.start, i.end)
                                   for i in ptr[:cnt.value]])
        ptr = C.POINTER(wp_comm_event)()
        cnt = C.c_int()
        check(lib.wp_trace_comm_events(self._h, C.byref(ptr), C.byref(cnt)))
        self.comm_events = [CommEvent(e.src_device, e.dst_device, e.post_time, e.arrival_time)
                            for e in ptr[:cnt.value]]

    def __del__(self):
        if getattr(self, "_owned", False) and self._h is not None and self._h.value:
            lib.wp_trace_free(self._h)
            self._h = None


def build_trace(intervals, comm_events=()) -> SimTrace:
    """wp_trace_build: a SimTrace from per-device interval lists (e.g. the
    measured traces of all ranks of a multi-process job merged), so
    bubble_ratio / memory_profile apply unchanged."""
    counts = (C.c_int * max(len(intervals), 1))(*[len(d) for d in intervals])
    flat = [iv for dev in intervals for iv in dev]
    ivs = (wp_interval * max(len(flat), 1))(*[
        wp_interval(i.action_index, int(i.kind), i.microbatch, i.slice_index, int(i.direction), i.start, i.end)
        for i in flat])
    evs = (wp_comm_event * max(len(comm_events), 1))(*[
        wp_comm_event(e.src_device, e.dst_device, e.post_time, e.arrival_time) for e in comm_events])
    h = C.c_void_p()
    check(lib.wp_trace_build(len(intervals), counts, ivs, len(comm_events), evs, C.byref(h)))
    return SimTrace(h)


def trace_to_gantt(trace: SimTrace, fmt: str = "svg") -> str:
    """trace_to_gantt (ref src/gantt.cpp:91-95): "svg" or "csv" text."""
    out = C.c_void_p()
    check(lib.wp_trace_to_gantt(trace._h, fmt.encode(), C.byref(out)))
    try:
        return C.string_at(out).decode()
    finally:
        lib.wp_string_free(out)


def _compare_text(fn_args, fmt):
    out = C.c_void_p()
    check(fn_args(0 if fmt == "csv" else 1, C.byref(out)))
    try:
        return C.string_at(out).decode()
    finally:
        lib.wp_string_free(out)


def _requests(requests):
    reqs = [(Scheme(r[0]), int(r[1])) if isinstance(r, tuple) else (Scheme(r), 1) for r in requests]
    n = len(reqs)
    return n, (C.c_int * max(n, 1))(*[int(s) for s, _ in reqs]), (C.c_int * max(n, 1))(*[w for _, w in reqs])


def compare(requests, budget_devices, microbatches, cost: CostModel = None, fmt: str = "json") -> str:
    """compare + compare_to_json / compare_to_csv (ref src/analytics.cpp:221-331):
    requests are (Scheme, waves) pairs (or bare schemes, W=1) evaluated at one
    device budget; returns the reference's CSV or JSON text, rows in
    ascending makespan, failed rows last."""
    n, sch, wav = _requests(requests)
    k = (cost or CostModel())._c()
    return _compare_text(lambda f, o: lib.wp_compare(sch, wav, n, budget_devices, microbatches, C.byref(k), f, o),
                         fmt)


def compare_measured(requests, budget_devices, microbatches, traces, lists, t_comm=0.0, fmt: str = "json") -> str:
    """The same rows from measured traces (one per request, e.g. the GPU
    runtime's train_step traces of lists[i]): makespan in seconds, the
    bubble ratio of the measured trace, Hanayo's Eq. 1 at the measured mean
    slice costs and message latency t_comm."""
    n, sch, wav = _requests(requests)
    tr = (C.c_void_p * max(n, 1))(*[t._h for t in traces])
    ls = (C.c_void_p * max(n, 1))(*[x.handle for x in lists])
    return _compare_text(lambda f, o: lib.wp_compare_measured(sch, wav, n, budget_devices, microbatches, tr, ls,
                                                              float(t_comm), f, o), fmt)


def simulate(lst: ActionList, cost: CostModel = None) -> SimTrace:
    """simulate (ref src/simulate.cpp:57-178); raises ScheduleError on a stall."""
    cost = cost or CostModel()
    h = C.c_void_p()
    k = cost._c()
    check(lib.wp_simulate(lst.handle, C.byref(k), C.byref(h)))
    return SimTrace(h)


def bubble_ratio(trace: SimTrace) -> float:
    out = C.c_double()
    check(lib.wp_bubble_ratio(trace._h, C.byref(out)))
    return out.value


def memory_profile(trace: SimTrace, lst: ActionList):
    """(weight_units, peak_activation_units) as lists of Fractions."""
    P = lst.config.devices
    w = (C.c_int64 * (2 * P))()
    pk = (C.c_int64 * (2 * P))()
    check(lib.wp_memory_profile(trace._h, lst.handle, w, pk))
    return ([Fraction(w[2 * d], w[2 * d + 1]) for d in range(P)],
            [Fraction(pk[2 * d], pk[2 * d + 1]) for d in range(P)])


def activation_variance(peaks) -> Fraction:
    n = len(peaks)
    if n == 0:
        return Fraction(0)
    mean = sum(peaks, Fraction(0)) / n
    return sum(((x - mean) ** 2 for x in peaks), Fraction(0)) / n


def analytic_bubble_hanayo(devices, waves, t_forward, t_backward, t_comm) -> Fraction:
    """Exact Eq. 1 (ref src/analytics.cpp:124-141); costs may be Fractions."""
    fr = [Fraction(x) for x in (t_forward, t_backward, t_comm)]
    arrs = [(C.c_int64 * 2)(f.numerator, f.denominator) for f in fr]
    out = (C.c_int64 * 2)()
    check(lib.wp_analytic_bubble_exact(devices, waves, arrs[0], arrs[1], arrs[2], out))
    return Fraction(out[0], out[1])


def analytic_bubble_hanayo_d(devices, waves, t_forward, t_backward, t_comm) -> float:
    out = C.c_double()
    check(lib.wp_analytic_bubble(devices, waves, t_forward, t_backward, t_comm, C.byref(out)))
    return out.value


def analytic_bubble_simplified(devices, waves) -> Fraction:
    out = (C.c_int64 * 2)()
    check(lib.wp_analytic_bubble_simplified(devices, waves, out))
    return Fraction(out[0], out[1])


def serialize_action_list(lst: ActionList) -> str:
    p = C.c_void_p()
    check(lib.wp_serialize(lst.handle, C.byref(p)))
    try:
        return C.string_at(p).decode()
    finally:
        lib.wp_string_free(p)


def parse_action_list(text: str) -> ActionList:
    h = C.c_void_p()
    check(lib.wp_parse(text.encode(), C.byref(h)))
    return ActionList(h)


def validate_all(lst: ActionList):
    """(ok, diagnostics text) -- validate_all (ref src/validate.cpp:529-536)."""
    ok = C.c_int()
    buf = C.create_string_buffer(1 << 16)
    check(lib.wp_validate(lst.handle, C.byref(ok), buf, len(buf)))
    return bool(ok.value), buf.value.decode()
