"""Host logic of the CUDA-IPC transport on CPU (no GPU needed): for every
generated list the static plan gives each message exactly one sender and
receiver, and each receiver at most two landing slots -- the transport's
memory on top of the reference's stash bound (src/analytics.cpp:61-76) --
because a slot is occupied only from its post (start of the compute before
the Receive, src/simulate.cpp:126) to its consumer's start."""
import ctypes as C

import pytest

import paper_2308_15762_b200 as wp
from paper_2308_15762_b200 import _native

lib = _native.lib
lib.wp_debug_ipc_plan.restype = C.c_int
lib.wp_debug_ipc_plan.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int]


def plan(lst):
    P = lst.config.devices
    slots = (C.c_int * P)()
    n = C.c_int()
    cap = 1 << 16
    msgs = (C.c_int * (3 * cap))()
    assert lib.wp_debug_ipc_plan(lst.handle, slots, C.byref(n), msgs, cap) == 0, lib.wp_last_error()
    return list(slots), [tuple(msgs[3 * i:3 * i + 3]) for i in range(n.value)]


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("W", [1, 2, 4])
@pytest.mark.parametrize("Bmul", [1, 2, 8])
def test_hanayo_landing_slots_at_most_two(P, W, Bmul):
    lst = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, P, Bmul * P, W))
    slots, msgs = plan(lst)
    sends = sum(1 for dev in lst.per_device for a in dev
                if a.kind in (wp.ActionKind.Send, wp.ActionKind.BatchedExchange))
    assert len(msgs) == sends                               # one entry per message
    assert all(1 <= s <= 2 for s in slots), slots
    for src, dst, slot in msgs:
        assert src != dst and 0 <= slot < slots[dst]
    # messages = 4 B W (P-1) for Hanayo
    assert len(msgs) == 4 * Bmul * P * W * (P - 1)


@pytest.mark.parametrize("scheme", [wp.Scheme.GPipe, wp.Scheme.Dapple])
def test_baseline_schemes_plan(scheme):
    lst = wp.generate_schedule(wp.make_config(scheme, 4, 8, 1))
    slots, msgs = plan(lst)
    assert max(slots) <= 2 and len(msgs) > 0


def test_single_device_has_no_messages():
    slots, msgs = plan(wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, 1, 4, 2)))
    assert slots == [0] and msgs == []
