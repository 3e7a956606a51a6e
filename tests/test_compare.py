"""compare / compare_to_csv / compare_to_json (ref src/analytics.cpp:221-331,
include/wavepipe/analytics.hpp:104-140) against the reference's own code.

Golden fixtures tests/golden/compare-p4-b8.{csv,json} were printed by
oracle/_ref/ref_driver (the reference's src/*.cpp compiled unchanged, see
oracle/Makefile):  ref_driver compare 4 8 1 2 0 csv|json gpipe:1 dapple:1
chimera:1 chimera-wave:2 hanayo:1 hanayo:2 hanayo:4.  When oracle/_ref is
built, more sweeps (failed rows, odd budgets, comm cost) are checked live.
"""
import json
import os
import subprocess

import pytest

import paper_2308_15762_b200 as wp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
REF = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
S = wp.Scheme
NAMES = {S.GPipe: "gpipe", S.Dapple: "dapple", S.Chimera: "chimera", S.ChimeraWave: "chimera-wave",
         S.Hanayo: "hanayo"}
SWEEP = [(S.GPipe, 1), (S.Dapple, 1), (S.Chimera, 1), (S.ChimeraWave, 2), (S.Hanayo, 1), (S.Hanayo, 2),
         (S.Hanayo, 4)]


@pytest.mark.parametrize("fmt", ["csv", "json"])
def test_compare_matches_reference_golden(fmt):
    with open(os.path.join(GOLD, f"compare-p4-b8.{fmt}")) as f:
        want = f.read()
    assert wp.compare(SWEEP, 4, 8, wp.CostModel(1, 2, 0), fmt=fmt) == want


def test_compare_rows_order_and_failures():
    rows = json.loads(wp.compare(SWEEP + [(S.Chimera, 2), (S.GPipe, 2)], 4, 8))
    ok = [r for r in rows if "error" not in r]
    assert [r["makespan"] for r in ok] == sorted(r["makespan"] for r in ok)
    assert all("error" in r for r in rows[len(ok):]) and len(rows) - len(ok) == 2
    assert rows[0]["scheme"] == "hanayo" and rows[0]["waves"] == 4
    assert wp.compare([], 4, 8, fmt="json") == "[]\n"


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("P,B,cost,reqs", [
    (4, 8, (1, 2, 0), SWEEP),
    (8, 16, (1, 2, 0.5), SWEEP + [(S.Hanayo, 3)]),
    (3, 6, (1, 3, 0), SWEEP),                      # odd budget: chimera / chimera-wave rows fail
    (2, 2, (2, 3, 1), [(S.Hanayo, 2), (S.GPipe, 2), (S.ChimeraWave, 1)]),
    (8, 64, (1, 2, 0), [(S.Hanayo, 1), (S.Hanayo, 2), (S.Hanayo, 4), (S.Dapple, 1), (S.Chimera, 1)]),
])
@pytest.mark.parametrize("fmt", ["csv", "json"])
def test_compare_matches_reference_live(P, B, cost, reqs, fmt):
    args = [REF, "compare", str(P), str(B)] + [repr(float(c)) for c in cost] + [fmt]
    args += [f"{NAMES[s]}:{w}" for s, w in reqs]
    want = subprocess.run(args, capture_output=True, text=True, check=True).stdout
    assert wp.compare(reqs, P, B, wp.CostModel(*cost), fmt=fmt) == want


def _row_list(req, P, B, cost):
    """The list and cost compare() evaluates for one request (chimera-wave:
    one of its two symmetric groups, ref src/analytics.cpp:236-247)."""
    scheme, W = req
    if scheme == S.ChimeraWave:
        cfg = wp.make_config(scheme, P // 2, B // 2, W, 2)
        cost = cost.rescaled(P, cfg.devices)
    else:
        cfg = wp.make_config(scheme, P, B, W)
    return wp.generate_schedule(cfg, cost), cost


@pytest.mark.parametrize("P,B,cost", [(4, 8, (1, 2, 0)), (8, 16, (1, 2, 0.5)), (4, 12, (2, 3, 0))])
@pytest.mark.parametrize("fmt", ["csv", "json"])
def test_compare_measured_on_simulated_traces_equals_compare(P, B, cost, fmt):
    """compare_measured -- the rows of MEASURED traces -- fed the simulator's
    traces of the same lists reproduces compare() byte for byte: the measured
    path shares the reference's row arithmetic, order and writers."""
    cm = wp.CostModel(*cost)
    lists, traces = [], []
    for req in SWEEP:
        lst, c = _row_list(req, P, B, cm)
        lists.append(lst)
        traces.append(wp.simulate(lst, c))
    got = wp.compare_measured(SWEEP, P, B, traces, lists, t_comm=cm.t_comm, fmt=fmt)
    assert got == wp.compare(SWEEP, P, B, cm, fmt=fmt)
