"""Bit-exact parity of the product schedule path with the reference (CPU).

Fixtures in tests/golden/ come from the reference's own code
(oracle/_ref/ref_driver, see tests/golden/make_golden.py):
  * the 5 byte-frozen goldens (proj/tests/data/*.json, acceptance criterion 10,
    proj/tests/acceptance.cpp:398-421) must regenerate byte-for-byte, and
    parse/serialize must round-trip byte-stably;
  * a grid of (scheme, P, B, W, costs) records: sha256 of the action streams,
    makespan, bubble, memory peaks/weights and Eq. 1 must match exactly.
"""
import gzip
import hashlib
import json
import os
from fractions import Fraction

import pytest

import paper_2308_15762_b200 as wp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = {"gpipe": wp.Scheme.GPipe, "dapple": wp.Scheme.Dapple, "chimera": wp.Scheme.Chimera,
         "chimera-wave": wp.Scheme.ChimeraWave, "hanayo": wp.Scheme.Hanayo}


def load_grid():
    with gzip.open(os.path.join(GOLDEN, "schedule_grid.json.gz"), "rt") as f:
        return json.load(f)


GRID = load_grid()


@pytest.mark.parametrize("name", ["gpipe-p4-b4", "dapple-p4-b4", "chimera-p4-b4", "hanayo-p4-b4-w1",
                                  "hanayo-p4-b4-w2"])
def test_golden_regenerates_byte_exact(name):
    text = open(os.path.join(GOLDEN, name + ".json")).read()
    stored = wp.parse_action_list(text)
    fresh = wp.generate_schedule(stored.config)
    assert wp.serialize_action_list(fresh) == text
    assert wp.serialize_action_list(stored) == text
    ok, report = wp.validate_all(stored)
    assert ok, report


@pytest.mark.parametrize("rec", GRID, ids=lambda r: f"{r['scheme']}-P{r['P']}-B{r['B']}-W{r['W']}-c{r['cost']}")
def test_grid_record(rec):
    cfg = wp.make_config(NAMES[rec["scheme"]], rec["P"], rec["B"], rec["W"])
    cost = wp.CostModel(*rec["cost"])
    lst = wp.generate_schedule(cfg, cost)
    assert hashlib.sha256(lst.compact().encode()).hexdigest() == rec["sha256"]
    if "actions" in rec:
        assert [[list(a) for a in dev] for dev in lst.per_device] == rec["actions"]
    tr = wp.simulate(lst, cost)
    assert tr.makespan == rec["makespan"]
    assert wp.bubble_ratio(tr) == rec["bubble"]
    weights, peaks = wp.memory_profile(tr, lst)
    assert [[p.numerator, p.denominator] for p in peaks] == rec["peaks"]
    assert [[w.numerator, w.denominator] for w in weights] == rec["weights"]
    assert len(tr.comm_events) == rec["n_comm_events"]
    if "intervals" in rec:
        got = [[[iv.action_index, int(iv.kind), iv.microbatch, iv.slice_index, iv.start, iv.end] for iv in dev]
               for dev in tr.intervals]
        assert got == rec["intervals"]
        assert [[e.src_device, e.dst_device, e.post_time, e.arrival_time] for e in tr.comm_events] == \
            rec["comm_events"]
    if "eq1" in rec:
        assert wp.analytic_bubble_hanayo_d(rec["P"], rec["W"], *rec["cost"]) == rec["eq1"]
    ok, report = wp.validate_all(lst)
    assert ok, report


def test_reference_unit_expectations():
    """Hand-derived values from the reference's own unit tests."""
    def make(s, P, B, W=1):
        lst = wp.generate_schedule(wp.make_config(s, P, B, W))
        return lst, wp.simulate(lst)
    # makespans 21/21/9/18/16 (proj/tests/test_simulate.cpp:53-65)
    assert make(wp.Scheme.GPipe, 4, 4)[1].makespan == 21
    assert make(wp.Scheme.Dapple, 4, 4)[1].makespan == 21
    assert make(wp.Scheme.Dapple, 1, 3)[1].makespan == 9
    assert make(wp.Scheme.Hanayo, 4, 4, 1)[1].makespan == 18
    assert make(wp.Scheme.Chimera, 4, 4)[1].makespan == 16
    # bubble 3/7, 1/3, 1/4 (proj/tests/test_analytics.cpp:50-62)
    assert abs(wp.bubble_ratio(make(wp.Scheme.GPipe, 4, 4)[1]) - 3 / 7) < 1e-12
    assert abs(wp.bubble_ratio(make(wp.Scheme.Hanayo, 4, 4, 1)[1]) - 1 / 3) < 1e-12
    assert abs(wp.bubble_ratio(make(wp.Scheme.Chimera, 4, 4)[1]) - 1 / 4) < 1e-12
    # Hanayo V-bottom: device 3 opens with F0.3, F0.4 (proj/tests/test_schedule.cpp:126-137)
    lst, _ = make(wp.Scheme.Hanayo, 4, 4, 1)
    comp = [(a.kind, a.microbatch, a.slice_index) for a in lst.per_device[3] if a.is_compute()]
    assert comp[:2] == [(wp.ActionKind.Forward, 0, 3), (wp.ActionKind.Forward, 0, 4)]
    # Dapple fusion: 12 BEs in 6 groups (proj/tests/test_schedule.cpp:185-205)
    lst, _ = make(wp.Scheme.Dapple, 4, 4)
    bes = [a for dev in lst.per_device for a in dev if a.kind == wp.ActionKind.BatchedExchange]
    assert len(bes) == 12 and len({a.batch_group for a in bes}) == 6
    # activation peaks Dapple [4,3,2,1], GPipe [4,4,4,4] (proj/tests/test_analytics.cpp:80-92)
    lst, tr = make(wp.Scheme.Dapple, 4, 4)
    assert wp.memory_profile(tr, lst)[1] == [4, 3, 2, 1]
    lst, tr = make(wp.Scheme.GPipe, 4, 4)
    assert wp.memory_profile(tr, lst)[1] == [4, 4, 4, 4]
    # variance 5/4 and 21/4 (proj/tests/test_analytics.cpp:94-100)
    for P, want in ((4, Fraction(5, 4)), (8, Fraction(21, 4))):
        lst, tr = make(wp.Scheme.Dapple, P, P)
        assert wp.activation_variance(wp.memory_profile(tr, lst)[1]) == want


def test_closed_forms():
    # acceptance criterion 1 (proj/tests/acceptance.cpp:81-97)
    for P in range(2, 65):
        for W in range(1, 9):
            assert wp.analytic_bubble_hanayo(P, W, 1, 2, 0) == wp.analytic_bubble_simplified(P, W)
    # point values (:99-114; proj/tests/test_analytics.cpp:163-186)
    assert wp.analytic_bubble_simplified(4, 1) == Fraction(2, 5)
    assert wp.analytic_bubble_simplified(4, 2) == Fraction(6, 27)
    assert wp.analytic_bubble_simplified(8, 1) == Fraction(14, 31)
    assert wp.analytic_bubble_simplified(8, 2) == Fraction(14, 55)
    assert wp.analytic_bubble_hanayo(4, 2, 1, 2, Fraction(1, 4)) == Fraction(61, 162)


def test_simulation_tracks_closed_form_and_waves_help():
    # acceptance criteria 4 and 6 (proj/tests/acceptance.cpp:130-186)
    prev = None
    for W in (1, 2, 4):
        lst = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, 4, 8, W))
        b = wp.bubble_ratio(wp.simulate(lst))
        if prev is not None:
            assert b < prev
        prev = b
        assert abs(b - float(wp.analytic_bubble_simplified(4, W))) <= 0.1


def test_config_errors():
    with pytest.raises(wp.ConfigError):
        wp.make_config(wp.Scheme.Hanayo, 4, 2, 2)  # B < P
    with pytest.raises(wp.ConfigError):
        wp.make_config(wp.Scheme.Dapple, 4, 4, 2)  # W>1 for a non-wave scheme
    with pytest.raises(wp.ConfigError):
        wp.make_config(wp.Scheme.Chimera, 3, 4)  # odd P
    with pytest.raises(wp.ConfigError):
        wp.parse_action_list('{"config": {}}')


def test_validator_catches_mutations():
    base = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, 4, 4, 2))
    streams = [list(dev) for dev in base.per_device]
    # drop a send
    for d, dev in enumerate(streams):
        for i, a in enumerate(dev):
            if a.kind == wp.ActionKind.Send:
                broken = [list(x) for x in streams]
                del broken[d][i]
                ok, report = wp.validate_all(wp.ActionList.from_actions(base.config, broken))
                assert not ok and "dependencies" in report
                break
        else:
            continue
        break
    # drop the flush
    broken = [dev[:-1] for dev in streams]
    ok, report = wp.validate_all(wp.ActionList.from_actions(base.config, broken))
    assert not ok and "flush" in report
    # duplicate a forward
    broken = [list(x) for x in streams]
    first = next(a for a in broken[0] if a.kind == wp.ActionKind.Forward)
    broken[0].insert(0, first)
    ok, report = wp.validate_all(wp.ActionList.from_actions(base.config, broken))
    assert not ok and "completeness" in report


def test_simulator_stall_raises():
    base = wp.generate_schedule(wp.make_config(wp.Scheme.Dapple, 2, 2))
    streams = [[a for a in dev if a.kind != wp.ActionKind.Send] for dev in base.per_device]
    lst = wp.ActionList.from_actions(base.config, streams)
    with pytest.raises(wp.ScheduleError):
        wp.simulate(lst)


def test_insert_comm_roundtrip():
    lst = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, 4, 8, 2))
    compute = [[a for a in dev if a.is_compute()] for dev in lst.per_device]
    again = wp.insert_comm(wp.ActionList.from_actions(lst.config, compute))
    assert again.compact() == lst.compact()


def test_deterministic():
    for s, P, B, W in ((wp.Scheme.Hanayo, 8, 64, 4), (wp.Scheme.Chimera, 8, 8, 1)):
        a = wp.generate_schedule(wp.make_config(s, P, B, W)).compact()
        b = wp.generate_schedule(wp.make_config(s, P, B, W)).compact()
        assert a == b
