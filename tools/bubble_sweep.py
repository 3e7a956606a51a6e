"""Theoretical bubble table for the BASELINE sweeps (CPU): the reference's
simulator on the generated list (CostModel 1/2/0 and at measured slice costs
if given) next to Eq. 1, for Hanayo W=1..4 at P=2/4/8 and the B sweep at
P=8 W=2.  Writes profiles/<round>_bubble_theory.md.

    python tools/bubble_sweep.py [r1]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_15762_b200 as wp  # noqa: E402

rnd = sys.argv[1] if len(sys.argv) > 1 else "r1"
rows = []
for P, B, W in [(p, 8, w) for p in (2, 4, 8) for w in (1, 2, 3, 4)] + [(8, b, 2) for b in (16, 24, 32, 48, 64)]:
    lst = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, P, B, W))
    sim = wp.simulate(lst)
    _, peaks = wp.memory_profile(sim, lst)
    msgs = sum(1 for d in lst.per_device for a in d if a.kind in (wp.ActionKind.Send, wp.ActionKind.BatchedExchange))
    rows.append((P, B, W, wp.bubble_ratio(sim), wp.analytic_bubble_hanayo_d(P, W, 1.0, 2.0, 0.0),
                 str(wp.analytic_bubble_simplified(P, W)), msgs, str(max(peaks))))
out = ["# Hanayo bubble: simulated (reference simulator on the generated list) vs Eq. 1",
       "", "CostModel T_F=1, T_B=2, T_C=0 (the goldens' cost model).  W=1 is the 1F1B-equivalent.",
       "Measured bubbles come from `bench.py` under torchrun (merged per-rank traces).", "",
       "| P | B | W | simulated | Eq. 1 | Eq. 1 simplified | messages / step | max stash peak (units) |",
       "|---|---|---|---|---|---|---|---|"]
out += [f"| {P} | {B} | {W} | {s:.4f} | {e:.4f} | {q} | {m} | {k} |" for P, B, W, s, e, q, m, k in rows]
os.makedirs("profiles", exist_ok=True)
with open(os.path.join("profiles", f"{rnd}_bubble_theory.md"), "w") as f:
    f.write("\n".join(out) + "\n")
print("\n".join(out))
