"""wp_trace_build: a trace assembled from per-device interval lists (how the
bench merges the measured traces of all ranks) must give the same
bubble_ratio / memory_profile as the trace it was taken from."""
import paper_2308_15762_b200 as wp


def test_rebuilt_trace_has_identical_metrics():
    for P, B, W in [(2, 4, 2), (4, 8, 2), (8, 8, 1), (3, 6, 3)]:
        lst = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, P, B, W))
        sim = wp.simulate(lst, wp.CostModel(1.0, 2.0, 0.05))
        rebuilt = wp.build_trace([list(d) for d in sim.intervals], sim.comm_events)
        assert rebuilt.makespan == sim.makespan
        assert wp.bubble_ratio(rebuilt) == wp.bubble_ratio(sim)
        assert wp.memory_profile(rebuilt, lst) == wp.memory_profile(sim, lst)
        assert rebuilt.comm_events == sim.comm_events


def test_merge_of_per_rank_parts():
    """Each rank contributes only its own device's intervals; the merge of
    the parts equals the whole."""
    lst = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, 4, 8, 2))
    sim = wp.simulate(lst)
    parts = [(sim.intervals[r], [e for e in sim.comm_events if e.src_device == r]) for r in range(4)]
    merged = wp.build_trace([p[0] for p in parts], [e for p in parts for e in p[1]])
    assert wp.bubble_ratio(merged) == wp.bubble_ratio(sim)
    assert sorted(merged.comm_events) == sorted(sim.comm_events)


def test_empty_trace():
    t = wp.build_trace([[], []])
    assert t.makespan == 0.0 and t.intervals == [[], []]
