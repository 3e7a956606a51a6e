"""End-to-end parity of the GPU runtime against the CPU oracle (GPU).

The pipelined step (any schedule, any placement) must equal sequential
gradient accumulation.  fp32 mode: loss and every parameter
gradient within 1e-5 relative (normwise per tensor) of an fp64 CPU run.
bf16 mode: within the tolerance stated in test_bf16_parity.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2308_15762_b200 as wp  # noqa: E402
from paper_2308_15762_b200.data import synthetic_batch  # noqa: E402
from oracle import model as om  # noqa: E402

TINY = dict(layers=4, hidden=256, heads=4, ffn=1024, seq=128, vocab=1024, micro_batch_size=2)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def build(desc, P, B, W, scheme=wp.Scheme.Hanayo, seed=7):
    cfg = wp.make_config(scheme, P, B, W)
    sched = wp.generate_schedule(cfg)
    rt = wp.Runtime(desc, sched, device_ids=[0] * P)
    params = om.init_params(desc, seed=seed)
    for name, t in params.items():
        rt.set_param(name, t.numpy())
    return rt, params


def run_parity(desc, P, B, W, scheme=wp.Scheme.Hanayo, tol=1e-5):
    rt, params = build(desc, P, B, W, scheme)
    rt.set_update(False)
    tokens, labels = synthetic_batch(B, desc.micro_batch_size, desc.seq, desc.vocab, causal=desc.causal)
    loss = rt.train_step(tokens, labels)
    ref_loss, ref_grads = om.reference_step(params, tokens, labels, desc)
    assert abs(loss - ref_loss) <= tol * abs(ref_loss), (loss, ref_loss)
    worst = 0.0
    for name, g in ref_grads.items():
        got = rt.get_grad(name, g.numel())
        e = rel(got, g.numpy())
        worst = max(worst, e)
        assert e <= tol, f"{name}: normwise rel err {e:.3g} > {tol}"
    return loss, worst, rt


def test_fp32_tiny_hanayo_p4_w2_b8():
    """BASELINE config 1: tiny GPT, Hanayo P=4 W=2, 8 microbatches, fp32."""
    desc = wp.ModelDesc(**TINY, dtype="fp32")
    run_parity(desc, P=4, B=8, W=2)


@pytest.mark.parametrize("P,B,W", [(1, 4, 1), (2, 4, 1), (2, 4, 3), (4, 4, 1), (3, 6, 2), (8, 8, 2), (4, 8, 4)])
def test_fp32_schedules(P, B, W):
    desc = wp.ModelDesc(**dict(TINY, layers=2), dtype="fp32")
    run_parity(desc, P, B, W)


def test_fp32_bidirectional_untied():
    desc = wp.ModelDesc(**dict(TINY, layers=2), causal=False, tie_embeddings=False, dtype="fp32")
    run_parity(desc, P=2, B=4, W=2)


@pytest.mark.parametrize("scheme,P,B", [(wp.Scheme.Dapple, 2, 4), (wp.Scheme.GPipe, 2, 4)])
def test_fp32_baseline_schemes_untied(scheme, P, B):
    # classic placements split slice 0 and S-1 across devices: untied head
    desc = wp.ModelDesc(**dict(TINY, layers=2), tie_embeddings=False, dtype="fp32")
    run_parity(desc, P, B, 1, scheme=scheme)


@pytest.mark.parametrize("P,B,W", [(2, 4, 2), (4, 8, 1)])
def test_fp32_chimera_wave(P, B, W):
    """Chimera-wave (ref src/placement.cpp:79-80: Hanayo placement) runs on
    the in-process runtime like Hanayo: the V-shaped slices keep the
    embedding and the tied head on device 0."""
    desc = wp.ModelDesc(**dict(TINY, layers=2), dtype="fp32")
    run_parity(desc, P, B, W, scheme=wp.Scheme.ChimeraWave)


def test_fp32_sgd_and_adamw_update():
    for opt in ("sgd", "adamw"):
        desc = wp.ModelDesc(**dict(TINY, layers=1), dtype="fp32", optimizer=opt, lr=1e-2, weight_decay=0.01)
        rt, params = build(desc, 2, 4, 1)
        tokens, labels = synthetic_batch(4, desc.micro_batch_size, desc.seq, desc.vocab)
        rt.train_step(tokens, labels)
        _, g = om.reference_step(params, tokens, labels, desc)
        if opt == "sgd":
            want = om.sgd_update(params, g, desc.lr, desc.weight_decay)
        else:
            want = om.adamw_update(params, g, desc.lr, desc.beta1, desc.beta2, desc.eps, desc.weight_decay)
        for name, p0 in params.items():
            got = rt.get_param(name, p0.numel()).astype(np.float64)
            p = p0.double().numpy().ravel()
            w = want[name].numpy().ravel()
            if opt == "sgd":
                # fp32 storage of the updated parameter bounds the comparison:
                # one ulp of |p| on top of the update's own tolerance.
                tol = 1e-4 * np.abs(w - p).max() + 2.0 ** -22 * np.abs(w)
                assert np.all(np.abs(got - w) <= tol), (opt, name)
            else:
                # AdamW's first step is ~ lr * sign(g): exact where the gradient is
                # well above its own rounding noise, bounded by lr everywhere.
                gr = g[name].numpy().ravel()
                well = np.abs(gr) >= 1e-3 * np.sqrt(np.mean(gr ** 2))
                tol = 1e-3 * desc.lr + 2.0 ** -22 * np.abs(w)
                assert np.all(np.abs(got - w)[well] <= tol[well]), (opt, name)
                bound = desc.lr * (1.001 + desc.weight_decay * np.abs(p)) + 2.0 ** -22 * np.abs(p)
                assert np.all(np.abs(got - p) <= bound), (opt, name)


def test_bf16_parity():
    """bf16 tensor-core mode vs the fp64 oracle.  Stated tolerance: loss within
    1e-2 relative; per-tensor normwise gradient error within 5e-2 (bf16 inputs
    carry 2^-9 relative rounding per operand, accumulated over the stack)."""
    desc = wp.ModelDesc(**dict(TINY, layers=2), dtype="bf16")
    rt, params = build(desc, 2, 4, 2)
    rt.set_update(False)
    tokens, labels = synthetic_batch(4, desc.micro_batch_size, desc.seq, desc.vocab)
    loss = rt.train_step(tokens, labels)
    ref_loss, ref_grads = om.reference_step(params, tokens, labels, desc)
    assert abs(loss - ref_loss) <= 1e-2 * abs(ref_loss)
    for name, g in ref_grads.items():
        e = rel(rt.get_grad(name, g.numel()), g.numpy())
        assert e <= 5e-2, f"{name}: {e:.3g}"


@pytest.mark.parametrize("causal", [True, False])
def test_bf16_parity_head_dim_64(causal):
    """bf16 with 64-wide heads (the BERT-large / GPT2-medium head size) and
    seq 256 through the fused attention; same stated tolerance."""
    desc = wp.ModelDesc(layers=2, hidden=512, heads=8, ffn=2048, seq=256, vocab=2048, micro_batch_size=2,
                        causal=causal, dtype="bf16")
    rt, params = build(desc, 2, 4, 2)
    rt.set_update(False)
    tokens, labels = synthetic_batch(4, desc.micro_batch_size, desc.seq, desc.vocab, causal=causal)
    loss = rt.train_step(tokens, labels)
    ref_loss, ref_grads = om.reference_step(params, tokens, labels, desc)
    assert abs(loss - ref_loss) <= 1e-2 * abs(ref_loss)
    for name, g in ref_grads.items():
        e = rel(rt.get_grad(name, g.numel()), g.numpy())
        assert e <= 5e-2, f"{name}: {e:.3g}"


def test_measured_trace_and_launches():
    desc = wp.ModelDesc(**dict(TINY, layers=2), dtype="bf16")
    rt, _ = build(desc, 2, 4, 2)
    rt.set_tracing(True)
    tokens, labels = synthetic_batch(4, desc.micro_batch_size, desc.seq, desc.vocab)
    before = rt.launch_count()
    rt.train_step(tokens, labels)
    assert rt.launch_count() > before
    tr = rt.trace()
    sched = rt.schedule
    n_compute = sum(a.is_compute() for dev in sched.per_device for a in dev)
    assert sum(len(iv) for iv in tr.intervals) == n_compute
    assert tr.makespan > 0
    b = wp.bubble_ratio(tr)
    assert 0.0 <= b < 1.0
    for dev in tr.intervals:
        for iv in dev:
            assert iv.end >= iv.start >= 0.0
