"""Host-side pipeline logic on CPU: the executor contract of the runtime
(message keys, placement, partition, BE pairing, FIFO order) runs the action
list with the oracle's autograd compute and must reproduce sequential
gradient accumulation; plus the rendezvous-safety of every generated list for
an in-order point-to-point queue, and a gloo world_size=2 run."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

import paper_2308_15762_b200 as wp
from oracle import model as om
from oracle import pipeline as opl
from paper_2308_15762_b200.data import synthetic_batch


class Desc:
    layers, hidden, heads, ffn, seq, vocab, micro_batch_size = 2, 32, 2, 64, 8, 16, 2
    causal, tie_embeddings = True, True


def schedule(P, B, W, scheme=wp.Scheme.Hanayo):
    lst = wp.generate_schedule(wp.make_config(scheme, P, B, W))
    acts = [[tuple(int(x) for x in a) for a in dev] for dev in lst.per_device]
    return acts, lst.placement


def close(devs_grads, ref):
    for name, g in ref.items():
        got = devs_grads[name]
        assert torch.allclose(got, g, rtol=1e-10, atol=1e-12), name


def collect(devs):
    out = {}
    for dv in devs:
        for name, p in dv.P.items():
            if p.grad is not None:
                out[name] = out.get(name, 0) + p.grad
    return out


@pytest.mark.parametrize("P,B,W", [(1, 2, 2), (2, 4, 2), (4, 4, 1), (3, 6, 2), (4, 8, 2)])
def test_local_interpreter_equals_sequential(P, B, W):
    d = Desc()
    params = om.init_params(d, seed=5)
    tokens, labels = synthetic_batch(B, d.micro_batch_size, d.seq, d.vocab)
    acts, pl = schedule(P, B, W)
    devs = opl.run_local(d, params, acts, pl, B, tokens, labels)
    ref_loss, ref = om.reference_step(params, tokens, labels, d)
    assert abs(sum(dv.loss for dv in devs) - ref_loss) < 1e-10
    close(collect(devs), ref)


def test_partition_matches_runtime_rules():
    d = Desc()
    us = opl.units(d)
    for P, W in ((1, 1), (1, 2), (2, 2), (4, 2), (8, 2), (8, 4)):
        lst = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, P, max(P, 2), W))
        S = lst.config.stages
        b = opl.partition(us, opl.slice_devices(lst.placement), P)
        assert b[0] == 0 and b[-1] == len(us)
        assert all(b[k] <= b[k + 1] for k in range(S))
        assert b[1] >= 1 or S == 1          # embedding in slice 0
        assert b[S - 1] <= len(us) - 1      # head in slice S-1


@pytest.mark.parametrize("scheme,W", [(wp.Scheme.Hanayo, 1), (wp.Scheme.Hanayo, 2), (wp.Scheme.Hanayo, 4),
                                      (wp.Scheme.Dapple, 1), (wp.Scheme.Chimera, 1)])
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_channel_plan_covers_every_message(scheme, W, P):
    """Sender-order channels (the oracle interpreter's receive plan, gloo
    point-to-point) deliver each incoming message of every device exactly
    once, from the right peer."""
    if scheme == wp.Scheme.Chimera and P % 2:
        return
    lst = wp.generate_schedule(wp.make_config(scheme, P, 2 * P, W))
    acts = [[tuple(int(x) for x in a) for a in dev] for dev in lst.per_device]
    ch = opl.channels(acts)
    for d in range(P):
        planned = sorted((src, k) for (src, dst), ks in ch.items() if dst == d for k in ks)
        assert planned == sorted(opl.incoming(acts, d))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = Desc()
        B = 4
        params = om.init_params(d, seed=9)
        tokens, labels = synthetic_batch(B, d.micro_batch_size, d.seq, d.vocab)
        acts, pl = schedule(world, B, 2)
        dev = opl.run_dist(d, params, acts, pl, B, tokens, labels)
        ref_loss, ref = om.reference_step(params, tokens, labels, d)
        ok = True
        for name, p in dev.P.items():
            if p.grad is None:
                continue
            ok &= bool(torch.allclose(p.grad, ref[name], rtol=1e-10, atol=1e-12))
        losses = [None] * world
        dist.all_gather_object(losses, dev.loss)
        ok &= abs(sum(losses) - ref_loss) < 1e-10
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in range(2))
    assert results == {0: True, 1: True}


def _dp_worker(rank, world, P, D, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = Desc()
        B = 4
        params = om.init_params(d, seed=13)
        replica = rank // P
        tokens, labels = synthetic_batch(B * D, d.micro_batch_size, d.seq, d.vocab)
        mine = slice(B * replica, B * (replica + 1))
        acts, pl = schedule(P, B, 2)
        dev = opl.run_dist(d, params, acts, pl, B, tokens[mine], labels[mine], replicas=D)
        ref_loss, ref = om.reference_step(params, tokens, labels, d)
        ok = True
        for name, p in dev.P.items():
            if p.grad is not None:
                ok &= bool(torch.allclose(p.grad, ref[name], rtol=1e-10, atol=1e-12))
        losses = [None] * world
        dist.all_gather_object(losses, dev.loss)
        # each rank holds its share of the replica-averaged loss
        ok &= abs(sum(losses) - ref_loss) < 1e-10
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_gloo_data_parallel_replicas():
    """P=2 pipeline devices x D=2 replicas (4 gloo processes, the runtime's
    rank layout): replica-averaged gradients equal sequential accumulation
    over all 2B microbatches."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    P, D = 2, 2
    procs = [ctx.Process(target=_dp_worker, args=(r, P * D, P, D, port, q)) for r in range(P * D)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    results = dict(q.get(timeout=5) for _ in range(P * D))
    assert results == {r: True for r in range(P * D)}
