"""trace_to_gantt (ref src/gantt.cpp:91-95): the SVG and CSV renderings of
each golden schedule's simulated trace are byte-identical to the reference's
own renderer (fixtures frozen by tests/golden/make_golden.py from
oracle/_ref), and the same call renders a measured-style trace."""
import os

import pytest

import paper_2308_15762_b200 as wp

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDENS = ["gpipe-p4-b4", "dapple-p4-b4", "chimera-p4-b4", "hanayo-p4-b4-w1", "hanayo-p4-b4-w2"]


@pytest.mark.parametrize("name", GOLDENS)
@pytest.mark.parametrize("fmt", ["csv", "svg"])
def test_gantt_matches_reference(name, fmt):
    lst = wp.parse_action_list(open(os.path.join(HERE, "golden", name + ".json")).read())
    got = wp.trace_to_gantt(wp.simulate(lst), fmt)
    want = open(os.path.join(HERE, "golden", "gantt", f"{name}.{fmt}")).read()
    assert got == want


def test_gantt_of_built_trace_and_bad_format():
    iv = wp.TraceInterval(0, wp.ActionKind.Forward, 0, 0, wp.Direction.Down, 0.0, 0.002)
    tr = wp.build_trace([[iv], []])
    csv = wp.trace_to_gantt(tr, "csv")
    assert csv.splitlines() == ["device,kind,microbatch,slice,start,end", "0,forward,0,0,0,0.002"]
    with pytest.raises(wp.ConfigError):
        wp.trace_to_gantt(tr, "png")
