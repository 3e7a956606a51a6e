"""Multi-process pipeline on the GPU: one process per pipeline device, the
CUDA-IPC transport (copy-engine pushes into IPC-mapped landing slots,
stream-memory-op flags), gloo for the handle exchange only (GPU).

On a 1-GPU box every rank maps to cuda:0 (CUDA IPC works between processes
on one device), so the multi-process path -- handle exchange, slot layout,
arrival/free flags, epoch reuse across steps -- is exercised exactly as on
8 GPUs; only the bytes do not cross NVLink.

Checks: fp32 loss and per-parameter gradients equal the single-process
run of the same list (same kernels, same per-device order; within 1e-6
normwise, the float atomics of the reductions are the only difference) and
the fp64 CPU oracle within 1e-5; three updating bf16 AdamW steps reproduce
the single-process loss trajectory within 1e-3 (slot reuse across epochs).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

TINY = dict(layers=2, hidden=256, heads=4, ffn=1024, seq=128, vocab=1024, micro_batch_size=2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _desc(dtype, optimizer="sgd", tie=True):
    import json
    import paper_2308_15762_b200 as wp
    widths = json.loads(os.environ["WP_TEST_WIDTHS"]) if os.environ.get("WP_TEST_WIDTHS") else TINY
    return wp.ModelDesc(**widths, dtype=dtype, optimizer=optimizer, lr=1e-3, weight_decay=0.01, tie_embeddings=tie)


def _run(rt, params, B, desc, steps, update, replica=0):
    from paper_2308_15762_b200.data import synthetic_batch
    for name, t in params.items():
        try:
            rt.set_param(name, t.numpy())
        except Exception:  # parameter owned by another rank
            pass
    rt.set_update(update)
    tokens, labels = synthetic_batch(B * (replica + 1), desc.micro_batch_size, desc.seq, desc.vocab)
    tokens, labels = tokens[B * replica:], labels[B * replica:]  # replica r: microbatches [rB, (r+1)B)
    losses = [rt.train_step(tokens, labels) for _ in range(steps)]
    grads = {n: rt.get_grad(n, k) for n, k in rt.param_names()}
    return losses, grads


def _worker(rank, world, port, B, W, dtype, optimizer, steps, update, q, D=1, scheme="Hanayo"):
    import faulthandler
    import sys
    import torch.distributed as dist
    faulthandler.dump_traceback_later(150, exit=True, file=sys.stderr)  # a hang fails loudly
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2308_15762_b200 as wp
        from oracle import model as om
        ngpu = torch.cuda.device_count()
        dev = rank % ngpu
        torch.cuda.set_device(dev)
        desc = _desc(dtype, optimizer, tie=scheme not in ("GPipe", "Dapple"))
        P = world // D
        sched = wp.generate_schedule(wp.make_config(getattr(wp.Scheme, scheme), P, B, W, D))
        rt = wp.Runtime(desc, sched, transport=wp.TRANSPORT_IPC, device_ids=[dev], rank=rank)
        ok, why = rt.ipc_status()
        assert ok, why  # the set-up probe of every mapped peer (copy + stream-op write)
        params = om.init_params(desc, seed=21)
        replica = rank // P
        losses, grads = _run(rt, params, B, desc, steps, update, replica=replica)
        # landing slots are reused as soon as the consumer copied them out:
        # at most two per GPU for the generated lists
        msg = desc.micro_batch_size * desc.seq * desc.hidden * (4 if dtype == "fp32" else 2)
        _, landing = rt.memory()
        assert landing <= 2 * ((msg + 255) // 256 * 256), (landing, msg)
        _check_stash(wp, rt, sched, rank % P)
        all_losses = [None] * world
        dist.all_gather_object(all_losses, losses)
        rt.close()
        # loss: sum over the pipeline devices of a replica, mean over replicas
        q.put((rank, [sum(x) / D for x in zip(*all_losses)], grads))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


def _check_stash(wp, rt, sched, pipe):
    """This rank's activation stash follows the reference's liveness and
    stays within memory_profile's peak units x bytes per unit (ref
    src/analytics.cpp:48-91; a slice's unit fraction from the placement)."""
    from fractions import Fraction
    peak, per_slice = rt.stash(pipe)
    live = best = 0
    for a in sched.per_device[pipe]:
        if a.kind == wp.ActionKind.Forward:
            live += per_slice[a.slice_index]
            best = max(best, live)
        elif a.kind == wp.ActionKind.Backward:
            live -= per_slice[a.slice_index]
    assert peak == best, (pipe, peak, best)
    cfg = sched.config
    if not any(per_slice):  # every slice of this device is empty (S > units)
        assert peak == 0
        return
    if cfg.scheme == wp.Scheme.Hanayo:
        _, peaks = wp.memory_profile(wp.simulate(sched, wp.CostModel(1.0, 2.0, 0.0)), sched)
        unit = max(Fraction(b) * 2 * cfg.waves for b in per_slice if b)
        assert peak <= peaks[pipe] * unit, (pipe, peak, float(peaks[pipe] * unit))


def _stall_worker(rank, world, port, q):
    """Rank 1 connects but never steps: rank 0's step must fail with the
    stall error naming its blocked action, then free cleanly."""
    import faulthandler
    import sys
    import torch.distributed as dist
    faulthandler.dump_traceback_later(150, exit=True, file=sys.stderr)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import time
        import paper_2308_15762_b200 as wp
        from paper_2308_15762_b200.data import synthetic_batch
        torch.cuda.set_device(0)
        desc = _desc("fp32")
        sched = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, 2, 4, 2))
        rt = wp.Runtime(desc, sched, transport=wp.TRANSPORT_IPC, device_ids=[0], rank=rank, stall_timeout=3.0)
        result = "idle"
        if rank == 0:
            tokens, labels = synthetic_batch(4, desc.micro_batch_size, desc.seq, desc.vocab)
            t0 = time.time()
            try:
                rt.train_step(tokens, labels)
                result = "no error"
            except wp.ScheduleError as e:
                result = (e.code, str(e), time.time() - t0)
            try:
                rt.train_step(tokens, labels)
                result = "second step ran"
            except wp.ScheduleError:
                pass
            rt.close()  # must not hang: the stalled waits were released
        dist.barrier()
        if rank == 1:
            rt.close()
        q.put((rank, result))
    except Exception as e:
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_stall_watchdog_names_blocked_action():
    """Executor contract, stall row (ref src/simulate.cpp:160-165): a peer that
    never runs its program makes the step return error code 1 (semantic,
    the reference's SimulationError) within the stall timeout, naming the
    action this rank is blocked at -- not a hang."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stall_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(2):
            r, res = q.get(timeout=200)
            out[r] = res
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert isinstance(out[0], tuple), out
    code, msg, waited = out[0]
    assert code == 1, out[0]
    assert "stalled" in msg and "blocked at" in msg and "device 0" in msg, msg
    assert 2.5 <= waited < 60, waited
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def _spawn(world, B, W, dtype, optimizer="sgd", steps=1, update=False, D=1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, W, dtype, optimizer, steps, update, q, D))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(world):
            rank, losses, grads = q.get(timeout=200)
            out[rank] = (losses, grads)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    for r, (losses, grads) in out.items():
        assert grads is not None, f"rank {r} failed: {losses}"
    losses = out[0][0]
    grads = {}
    for _, g in out.values():
        grads.update(g)
    return losses, grads


def _spawn_raw(world, B, W, dtype, optimizer="sgd", steps=1, update=False, D=1, scheme="Hanayo"):
    """Per-rank (losses, grads) of a spawned job."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, W, dtype, optimizer, steps, update, q, D, scheme))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(world):
            rank, losses, grads = q.get(timeout=200)
            assert grads is not None, f"rank {rank} failed: {losses}"
            out[rank] = (losses, grads)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    return out


def _single_process(world, B, W, dtype, optimizer="sgd", steps=1, update=False):
    import paper_2308_15762_b200 as wp
    from oracle import model as om
    desc = _desc(dtype, optimizer)
    sched = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, world, B, W))
    rt = wp.Runtime(desc, sched, device_ids=[0] * world)
    params = om.init_params(desc, seed=21)
    losses, grads = _run(rt, params, B, desc, steps, update)
    rt.close()
    return losses, grads, params


@pytest.mark.parametrize("world,B,W", [(2, 4, 2), (4, 8, 2), (3, 6, 1), (8, 8, 2)])
def test_ipc_fp32_equals_single_process_and_oracle(world, B, W):
    from oracle import model as om
    from paper_2308_15762_b200.data import synthetic_batch
    losses, grads = _spawn(world, B, W, "fp32")
    ref_losses, ref_grads, params = _single_process(world, B, W, "fp32")
    assert abs(losses[0] - ref_losses[0]) <= 1e-6 * abs(ref_losses[0])
    assert set(grads) == set(ref_grads)
    for n in ref_grads:
        a, b = grads[n].astype(np.float64), ref_grads[n].astype(np.float64)
        assert np.linalg.norm(a - b) <= 1e-6 * max(np.linalg.norm(b), 1e-30), n
    desc = _desc("fp32")
    tokens, labels = synthetic_batch(B, desc.micro_batch_size, desc.seq, desc.vocab)
    want_loss, want = om.reference_step(params, tokens, labels, desc)
    assert abs(losses[0] - want_loss) <= 1e-5 * abs(want_loss)
    for n, g in want.items():
        w = g.numpy().ravel().astype(np.float64)
        e = np.linalg.norm(grads[n] - w) / max(np.linalg.norm(w), 1e-30)
        assert e <= 1e-5, (n, e)


def test_ipc_bf16_adamw_three_steps_follow_single_process():
    """Landing slots are reused every step (epoch-tagged flags): three
    updating bf16 steps follow the single-process loss trajectory."""
    losses, _ = _spawn(2, 4, 2, "bf16", optimizer="adamw", steps=3, update=True)
    ref, _, _ = _single_process(2, 4, 2, "bf16", optimizer="adamw", steps=3, update=True)
    assert np.allclose(losses, ref, rtol=1e-3, atol=0), (losses, ref)
    assert losses[2] < losses[0]


@pytest.mark.parametrize("P,D,B,W", [(1, 2, 4, 2), (2, 2, 4, 2), (1, 3, 2, 1)])
def test_data_parallel_replicas_equal_sequential_big_batch(P, D, B, W):
    """D replicas x P pipeline devices (rank = replica*P + device): replica r
    runs microbatches [rB, (r+1)B); the peer-memory all-reduce at the
    optimizer step averages the gradients, so every replica holds the
    gradient of sequential accumulation over all D*B microbatches (fp32,
    1e-5 vs the fp64 oracle) -- the same in every replica."""
    from oracle import model as om
    from paper_2308_15762_b200.data import synthetic_batch
    world = P * D
    out = _spawn_raw(world, B, W, "fp32", D=D)
    desc = _desc("fp32")
    params = om.init_params(desc, seed=21)
    tokens, labels = synthetic_batch(B * D, desc.micro_batch_size, desc.seq, desc.vocab)
    want_loss, want = om.reference_step(params, tokens, labels, desc)
    assert abs(out[0][0][0] - want_loss) <= 1e-5 * abs(want_loss)
    for rank, (_, grads) in out.items():
        for n, g in grads.items():
            w = want[n].numpy().ravel().astype(np.float64)
            e = np.linalg.norm(g - w) / max(np.linalg.norm(w), 1e-30)
            assert e <= 1e-5, (rank, n, e)
    # replicas hold bit-identical gradients (one summation order for all)
    for rank, (_, grads) in out.items():
        for n, g in grads.items():
            assert np.array_equal(g, out[rank % P][1][n]), (rank, n)


def test_data_parallel_bf16_adamw_steps():
    losses = _spawn_raw(2, 4, 2, "bf16", optimizer="adamw", steps=3, update=True, D=2)[0][0]
    assert losses[2] < losses[0]


@pytest.mark.parametrize("P,D,B", [(2, 1, 4), (4, 1, 8), (2, 2, 4)])
def test_chimera_mirrored_stages_equal_oracle(P, D, B):
    """Chimera (the reference's bidirectional baseline, src/placement.cpp:41-50):
    device p holds stage p for the down pipeline and stage P-1-p for the up
    one, so devices p and P-1-p hold the same stages and their gradients are
    summed over peer memory at the optimizer step (with the D replicas, then
    scaled by 1/D).  fp32 loss and every gradient equal the fp64 oracle's
    sequential step over the D*B microbatches, bit-identical on all holders."""
    from oracle import model as om
    from paper_2308_15762_b200.data import synthetic_batch
    out = _spawn_raw(P * D, B, 1, "fp32", D=D, scheme="Chimera")
    desc = _desc("fp32")
    params = om.init_params(desc, seed=21)
    tokens, labels = synthetic_batch(B * D, desc.micro_batch_size, desc.seq, desc.vocab)
    want_loss, want = om.reference_step(params, tokens, labels, desc)
    assert abs(out[0][0][0] - want_loss) <= 1e-5 * abs(want_loss)
    for rank, (_, grads) in out.items():
        for n, g in grads.items():
            w = want[n].numpy().ravel().astype(np.float64)
            e = np.linalg.norm(g - w) / max(np.linalg.norm(w), 1e-30)
            assert e <= 1e-5, (rank, n, e)
        mirror = (rank // P) * P + P - 1 - rank % P
        for n, g in grads.items():
            assert np.array_equal(g, out[mirror][1][n]), (rank, n)


def test_chimera_needs_ipc_transport():
    import paper_2308_15762_b200 as wp
    sched = wp.generate_schedule(wp.make_config(wp.Scheme.Chimera, 2, 4))
    with pytest.raises(Exception, match="IPC transport"):
        wp.Runtime(_desc("fp32"), sched, device_ids=[0, 0])


@pytest.mark.parametrize("scheme,P,B", [("Dapple", 4, 8), ("GPipe", 2, 4)])
def test_classic_schemes_over_ipc_equal_oracle(scheme, P, B):
    """The baseline schemes (classic placement, src/placement.cpp:32-38; the
    head on the last device, so untied) through the same IPC transport."""
    from oracle import model as om
    from paper_2308_15762_b200.data import synthetic_batch
    out = _spawn_raw(P, B, 1, "fp32", scheme=scheme)
    desc = _desc("fp32", tie=False)
    params = om.init_params(desc, seed=21)
    tokens, labels = synthetic_batch(B, desc.micro_batch_size, desc.seq, desc.vocab)
    want_loss, want = om.reference_step(params, tokens, labels, desc)
    assert abs(out[0][0][0] - want_loss) <= 1e-5 * abs(want_loss)
    for rank, (_, grads) in out.items():
        for n, g in grads.items():
            w = want[n].numpy().ravel().astype(np.float64)
            e = np.linalg.norm(g - w) / max(np.linalg.norm(w), 1e-30)
            assert e <= 1e-5, (rank, n, e)


def test_measured_compare_tool_two_ranks():
    """tools/compare_measured.py on two ranks sharing the GPU (functional):
    every scheme that runs at P=2 yields a measured row (seconds, bubble in
    [0, 1)), in the reference's CSV layout, sorted by makespan."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WP_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", f"--master-port={_free_port()}", os.path.join(root, "tools", "compare_measured.py"),
           "--model", "tiny-gpt", "--mbs", "2", "--microbatches", "4"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = out.stdout.strip().splitlines()
    assert lines[0].startswith("scheme,devices,microbatches,waves,makespan,simulated_bubble_ratio")
    rows = [ln.split(",") for ln in lines[1:]]
    names = {(r[0], r[3]) for r in rows}
    assert {("gpipe", "1"), ("dapple", "1"), ("chimera", "1"), ("hanayo", "1"), ("hanayo", "2")} <= names
    spans = [float(r[4]) for r in rows if r[4]]
    assert spans == sorted(spans) and all(0 < s < 60 for s in spans)
    assert all(0.0 <= float(r[5]) < 1.0 for r in rows if r[5])


def test_ipc_bf16_gpt2_medium_widths_equal_oracle():
    """Two processes over CUDA IPC at the GPT2-medium widths (BASELINE
    config 2's layer shapes, d=64 heads), Hanayo P=2 W=2, bf16: loss and
    every gradient against the bf16 rounding-point oracle (1e-2 normwise,
    the stated bf16 tolerance), messages of mbs x seq x hidden bf16."""
    import json
    from oracle import model as om
    from paper_2308_15762_b200.data import synthetic_batch
    widths = dict(layers=2, hidden=1024, heads=16, ffn=4096, seq=512, vocab=50304, micro_batch_size=1)
    os.environ["WP_TEST_WIDTHS"] = json.dumps(widths)
    try:
        losses, grads = _spawn(2, 4, 2, "bf16")
        desc = _desc("fp32")
    finally:
        del os.environ["WP_TEST_WIDTHS"]
    params = om.init_params(desc, seed=21)
    tokens, labels = synthetic_batch(4, 1, widths["seq"], widths["vocab"])
    want_loss, want = om.reference_step(params, tokens, labels, desc, emulate="bf16")
    assert abs(losses[0] - want_loss) <= 2e-3 * abs(want_loss), (losses[0], want_loss)
    for n, g in want.items():
        w = g.numpy().ravel().astype(np.float64)
        e = np.linalg.norm(grads[n].astype(np.float64) - w) / max(np.linalg.norm(w), 1e-30)
        assert e <= 1e-2, (n, e)
