"""Pin the oracles before trusting them (CPU).

* oracle/schedule.py (pure-Python restatement) against the reference's 5
  byte-frozen goldens and the small oracle/_ref grid records.
* oracle/model.py (torch CPU) basic invariants: initial loss ~ ln V, autograd
  gradients vs central finite differences on a few coordinates.
"""
import gzip
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import model as om
from oracle import schedule as osch
from paper_2308_15762_b200.data import synthetic_batch

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SCHEMES = {"gpipe": osch.GPIPE, "dapple": osch.DAPPLE, "chimera": osch.CHIMERA,
           "chimera-wave": osch.CHIMERA_WAVE, "hanayo": osch.HANAYO}
KIND = ["forward", "backward", "send", "receive", "batched_exchange", "optimizer_step"]


def golden_actions(name):
    doc = json.load(open(os.path.join(GOLDEN, name + ".json")))
    out = []
    for dev in doc["actions"]:
        row = []
        for a in dev:
            row.append((KIND.index(a["kind"]), a.get("microbatch", -1), a.get("local_module_rank", -1),
                        a.get("slice_index", -1), a.get("peer", -1),
                        {"activation": 0, "gradient": 1}.get(a.get("payload"), -1), a.get("batch_group", -1)))
        out.append(row)
    return doc["config"], out


@pytest.mark.parametrize("name", ["gpipe-p4-b4", "dapple-p4-b4", "chimera-p4-b4", "hanayo-p4-b4-w1",
                                  "hanayo-p4-b4-w2"])
def test_python_oracle_matches_goldens(name):
    c, want = golden_actions(name)
    cfg = osch.make_config(SCHEMES[c["scheme"]], c["P"], c["B"], c["W"], c["D"])
    got, pl = osch.generate_schedule(cfg)
    assert got == want
    mk, iv, ev = osch.simulate(cfg, got)
    assert mk == {"gpipe-p4-b4": 21, "dapple-p4-b4": 21, "chimera-p4-b4": 16, "hanayo-p4-b4-w1": 18,
                  "hanayo-p4-b4-w2": 15.25}[name]  # proj/tests/data/README.md:37-39


def small_records():
    with gzip.open(os.path.join(GOLDEN, "schedule_grid.json.gz"), "rt") as f:
        recs = json.load(f)
    return [r for r in recs if "actions" in r and r["P"] * r["B"] * r["W"] <= 96]


@pytest.mark.parametrize("rec", small_records(),
                         ids=lambda r: f"{r['scheme']}-P{r['P']}-B{r['B']}-W{r['W']}-c{r['cost']}")
def test_python_oracle_matches_ref_grid(rec):
    cfg = osch.make_config(SCHEMES[rec["scheme"]], rec["P"], rec["B"], rec["W"])
    got, pl = osch.generate_schedule(cfg, tuple(rec["cost"]))
    assert [[list(a) for a in dev] for dev in got] == rec["actions"]
    mk, iv, ev = osch.simulate(cfg, got, tuple(rec["cost"]))
    assert mk == rec["makespan"]
    assert osch.bubble_ratio(mk, iv) == rec["bubble"]
    _, peaks = osch.memory_profile(pl, iv)
    assert [[p.numerator, p.denominator] for p in peaks] == rec["peaks"]
    assert [list(e) for e in ev] == rec["comm_events"]


def test_python_oracle_closed_forms():
    for P in range(2, 20):
        for W in range(1, 6):
            assert osch.analytic_bubble_hanayo(P, W, 1, 2, 0) == osch.analytic_bubble_simplified(P, W)


class Desc:
    layers, hidden, heads, ffn, seq, vocab, micro_batch_size = 1, 16, 2, 32, 8, 32, 2
    causal, tie_embeddings = True, True


def test_model_oracle_initial_loss_and_fd_gradients():
    d = Desc()
    params = om.init_params(d, seed=3, nonzero_vectors=True)
    tokens, labels = synthetic_batch(2, d.micro_batch_size, d.seq, d.vocab)
    loss, grads = om.reference_step(params, tokens, labels, d)
    assert abs(loss - math.log(d.vocab)) < 0.5
    P64 = {k: v.double() for k, v in params.items()}

    def f(P):
        return sum(float(om.microbatch_loss(P, tokens[b], labels[b], d)) for b in range(2)) / 2

    g = torch.Generator().manual_seed(0)
    for name in ("wte", "h.0.attn.qkv.w", "h.0.ln2.b", "h.0.mlp.fc1.w", "lnf.w"):
        t = P64[name]
        for _ in range(3):
            i = int(torch.randint(t.numel(), (1,), generator=g))
            eps = 1e-6
            orig = t.view(-1)[i].item()
            t.view(-1)[i] = orig + eps
            fp = f(P64)
            t.view(-1)[i] = orig - eps
            fm = f(P64)
            t.view(-1)[i] = orig
            fd = (fp - fm) / (2 * eps)
            assert abs(fd - grads[name].view(-1)[i].item()) <= 1e-6 + 1e-5 * abs(fd)


def test_oracle_input_stream_matches_product():
    """oracle/data.py restates the SURVEY 8(d) input spec; it must produce the
    product's batches bit for bit (causal and bidirectional, several steps)."""
    from oracle import data as od
    from paper_2308_15762_b200 import data as pd
    for causal in (True, False):
        for step in (0, 3):
            a = od.synthetic_batch(3, 2, 64, 50304, causal=causal, step=step)
            b = pd.synthetic_batch(3, 2, 64, 50304, causal=causal, step=step)
            for x, y in zip(a, b):
                assert x.dtype == y.dtype and x.shape == y.shape and np.array_equal(x, y)
