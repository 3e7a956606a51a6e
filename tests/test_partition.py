"""Device-balanced slice partition of the runtime (host logic, CPU): cuts
are contiguous, the embedding stays in slice 0 and the LM head in slice S-1
(same Hanayo device, tied embeddings), and the busiest device's share is
close to 1/P -- at GPT-1.3B P=8 W=2 the equal-slice partition leaves the
head's device 1.5x loaded."""
import ctypes as C

import pytest

import paper_2308_15762_b200 as wp
from paper_2308_15762_b200 import _native

lib = _native.lib
lib.wp_debug_partition.restype = C.c_int
lib.wp_debug_partition.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double),
                                   C.POINTER(C.c_int)]

GPT13B = dict(layers=24, hidden=2048, heads=16, ffn=8192, seq=1024, vocab=50304, micro_batch_size=16, dtype="bf16")


def partition(desc, lst):
    S = lst.config.stages
    b = (C.c_int * (S + 1))()
    costs = (C.c_double * 4096)()
    n = C.c_int()
    d = desc._c()
    assert lib.wp_debug_partition(C.byref(d), lst.handle, b, costs, C.byref(n)) == 0, lib.wp_last_error()
    return list(b), list(costs[:n.value])


def device_loads(lst, b, costs):
    P = lst.config.devices
    load = [0.0] * P
    for d, slices in enumerate(lst.placement):
        for sl in slices:
            load[d] += sum(costs[b[sl]:b[sl + 1]])
    return load


@pytest.mark.parametrize("P,W,bound", [(2, 2, 1.05), (4, 2, 1.05), (8, 1, 1.06), (8, 2, 1.15), (8, 4, 1.06)])
def test_gpt13b_device_balance(P, W, bound):
    desc = wp.ModelDesc(**GPT13B)
    lst = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, P, 8, W))
    b, costs = partition(desc, lst)
    S = lst.config.stages
    assert b[0] == 0 and b[-1] == len(costs) and all(b[k] <= b[k + 1] for k in range(S))
    assert b[1] >= 1 and b[S - 1] <= len(costs) - 1      # embedding in slice 0, head in slice S-1
    load = device_loads(lst, b, costs)
    assert max(load) / (sum(load) / P) <= bound, load


def test_tiny_more_slices_than_units():
    desc = wp.ModelDesc(layers=4, hidden=256, heads=4, ffn=1024, seq=128, vocab=1024)
    lst = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, 4, 8, 2))  # S = 16 > 10 units
    b, costs = partition(desc, lst)
    assert b[0] == 0 and b[-1] == len(costs) and all(b[k] <= b[k + 1] for k in range(16))


@pytest.mark.parametrize("P,W", [(1, 2), (2, 2), (4, 2), (8, 2), (8, 4), (3, 1)])
@pytest.mark.parametrize("model", ["gpt13b", "tiny"])
def test_oracle_restates_runtime_partition(P, W, model):
    """oracle/pipeline.py's partition (the CPU interpreter's slices) equals
    the runtime's device-balanced cut bit for bit."""
    from oracle import pipeline as op
    desc = wp.ModelDesc(**GPT13B) if model == "gpt13b" else wp.ModelDesc(layers=4, hidden=256, heads=4, ffn=1024,
                                                                          seq=128, vocab=1024)
    lst = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, P, 8, W))
    b, _ = partition(desc, lst)
    assert op.partition(op.units(desc), op.slice_devices(lst.placement), P) == b
