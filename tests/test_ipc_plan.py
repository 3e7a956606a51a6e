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


# ---------------------------------------------------------------------------
# Deadlock-freedom of the push protocol (ipc.cpp), modelled on CPU: compute c
# of device q starts once its remote input arrived; q posts message m at the
# start of the compute before its Receive (or at step begin); the sender's
# per-peer copy stream is FIFO in the receiver's issue order and pushes m
# once its producer ran and m is posted.  The runtime issues in CONSUMER
# order; sender program order is shown to deadlock Hanayo P=4 W=2 B=8.
F, BW, SEND, RECV, BE = 0, 1, 2, 3, 4


def _key(a):
    kind, mb, _, s, _, payload, _ = a
    out = kind in (SEND, BE)
    low = (s if out else s - 1) if payload == 0 else (s - 1 if out else s)
    return (payload, mb, low)


def _input_key(a):
    kind, mb, _, s = a[:4]
    return (0, mb, s - 1) if kind == F else (1, mb, s)


def _producer(key):
    payload, mb, low = key
    return (F, mb, low) if payload == 0 else (BW, mb, low + 1)


def _runs(lst, order):
    progs = [[tuple(int(x) for x in a) for a in dev] for dev in lst.per_device]
    P = len(progs)
    groups = {}
    for p, prog in enumerate(progs):
        for i, a in enumerate(prog):
            if a[0] == BE:
                groups.setdefault(a[6], []).append((p, i))
    src, post_at, consume_at, fifo = {}, {}, {}, {}
    computes = [[a for a in prog if a[0] in (F, BW)] for prog in progs]
    for q, prog in enumerate(progs):
        c, incoming = 0, []
        for i, a in enumerate(prog):
            if a[0] in (F, BW):
                c += 1
            elif a[0] == RECV:
                incoming.append(_key(a))
                src[_key(a)] = a[4]
            elif a[0] == BE:
                for p2, j in groups[a[6]]:
                    if p2 != q:
                        incoming.append(_key(progs[p2][j]))
                        src[_key(progs[p2][j])] = p2
            for k in incoming[len(post_at.get(q, {})):]:
                post_at.setdefault(q, {})[k] = c - 1
        cons = {_input_key(a): ci for ci, a in enumerate(computes[q])}
        for k in incoming:
            consume_at[(q, k)] = cons[k]
        for k in sorted(incoming, key=lambda k: cons[k]):
            fifo.setdefault((src[k], q), []).append(k)
    if order == "production":  # sender program order instead
        made = {}
        for p, prog in enumerate(progs):
            for i, a in enumerate(prog):
                if a[0] in (SEND, BE):
                    made[(p, _key(a))] = i
        fifo = {pq: sorted(ks, key=lambda k: made[(pq[0], k)]) for pq, ks in fifo.items()}
    started = [0] * P
    done_ops = set()  # (device, kind, mb, slice) computes that ran
    arrived = set()
    heads = {pq: 0 for pq in fifo}
    moved = True
    while moved:
        moved = False
        for (p, q), ks in fifo.items():
            while heads[(p, q)] < len(ks):
                k = ks[heads[(p, q)]]
                ready = (p,) + _producer(k) in done_ops
                posted = started[q] > post_at[q][k]
                if not (ready and posted):
                    break
                arrived.add((q, k))
                heads[(p, q)] += 1
                moved = True
        for q in range(P):
            while started[q] < len(computes[q]):
                a = computes[q][started[q]]
                k = _input_key(a)
                if (q, k) in consume_at and (q, k) not in arrived:
                    break
                done_ops.add((q, a[0], a[1], a[3]))
                started[q] += 1
                moved = True
    return all(started[q] == len(computes[q]) for q in range(P))


LISTS = ([(wp.Scheme.Hanayo, P, m * P, W) for P in (2, 4, 8) for W in (1, 2, 4) for m in (1, 2, 4)] +
         [(wp.Scheme.Chimera, P, m * P, 1) for P in (2, 4, 8) for m in (1, 2, 4)] +
         [(s, P, 2 * P, 1) for s in (wp.Scheme.GPipe, wp.Scheme.Dapple) for P in (2, 4, 8)])


@pytest.mark.parametrize("scheme,P,B,W", LISTS)
def test_push_protocol_in_consumer_order_never_deadlocks(scheme, P, B, W):
    lst = wp.generate_schedule(wp.make_config(scheme, P, B, W))
    assert _runs(lst, "consumer")



def test_production_order_fifo_deadlocks_hanayo():
    """The order the runtime used first (sender program order) stalls."""
    lst = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, 4, 8, 2))
    assert not _runs(lst, "production")
