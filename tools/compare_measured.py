"""Measured scheme comparison on the GPU runtime (f4: the reference's
`compare`, proj/src/analytics.cpp:221-331, over MEASURED traces).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        tools/compare_measured.py [--model gpt-1.3b-like] [--mbs 4] [--microbatches 8] [--fmt csv|json]

Every rank is one GPU (WP_BENCH_SHARE_GPU=1 maps all ranks to cuda:0: a
functional run, not a measurement).  For each scheme of the sweep (GPipe,
DAPPLE, Chimera, Chimera-wave, Hanayo W=1/2/4) at a device budget of N: the
list compare() would evaluate (chimera-wave as two symmetric groups of N/2,
the data-parallel D=2 of the reference's evaluation) runs on the IPC
transport for warm-up steps, then one traced step; the ranks' traces are put
on one device clock (%globaltimer) and merged, and rank 0 prints
wavepipe.compare_measured's rows: measured step time (s), measured bubble,
memory units, Eq. 1 at the measured slice costs and message latency.
Schemes that cannot run at this budget (odd N for Chimera, ...) come out
as failed rows, as in the reference.
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="gpt-1.3b-like")
    ap.add_argument("--mbs", type=int, default=4)
    ap.add_argument("--microbatches", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--fmt", default="csv", choices=["csv", "json"])
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    import bench
    import paper_2308_15762_b200 as wp
    from paper_2308_15762_b200.data import synthetic_batch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    share = os.environ.get("WP_BENCH_SHARE_GPU") == "1"
    dev = 0 if share else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo" if share else "nccl", **({} if share else {"device_id": torch.device("cuda", dev)}))
    S = wp.Scheme
    sweep = [(S.GPipe, 1), (S.Dapple, 1), (S.Chimera, 1), (S.ChimeraWave, 2), (S.Hanayo, 1), (S.Hanayo, 2),
             (S.Hanayo, 4)]
    m = bench.MODELS[args.model]
    B = args.microbatches
    reqs, traces, lists, comm = [], [], [], []
    for scheme, W in sweep:
        try:
            if scheme == S.ChimeraWave:
                cfg = wp.make_config(scheme, world // 2, B // 2, W, 2)
            else:
                cfg = wp.make_config(scheme, world, B, W)
            lst = wp.generate_schedule(cfg)
        except wp.ConfigError:
            continue  # compare() reports it as a failed row; nothing to measure
        P, D = cfg.devices, cfg.replicas
        desc = wp.ModelDesc(**m, micro_batch_size=args.mbs, tie_embeddings=scheme not in (S.GPipe, S.Dapple),
                            dtype="bf16", optimizer="adamw", lr=1e-4, weight_decay=0.01)
        rt = wp.Runtime(desc, lst, transport=wp.TRANSPORT_IPC, device_ids=[dev], rank=rank)
        tok, lab = synthetic_batch(cfg.microbatches, args.mbs, desc.seq, desc.vocab, step=rank // P)
        for _ in range(args.warmup):
            rt.train_step(tok, lab)
        rt.set_tracing(True)
        dist.barrier()
        rt.train_step(tok, lab)
        rt.set_tracing(False)
        tr = rt.trace()
        pipe = rank % P
        mine = (tr.intervals[pipe], [e for e in tr.comm_events if e.src_device == pipe], rt.step_clock_ns())
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        dist.barrier()
        rt.close()
        if rank == 0:
            t0 = min(p[2] for p in parts[:P])
            off = [(p[2] - t0) * 1e-9 for p in parts[:P]]
            merged = wp.build_trace(
                [[iv._replace(start=iv.start + off[d], end=iv.end + off[d]) for iv in parts[d][0]] for d in range(P)],
                [e._replace(post_time=e.post_time + off[d], arrival_time=e.arrival_time + off[d])
                 for d in range(P) for e in parts[d][1]])
            reqs.append((scheme, W))
            traces.append(merged)
            lists.append(lst)
            comm += [e.arrival_time - e.post_time for e in merged.comm_events]
    if rank == 0:
        t_comm = statistics.mean(comm) if comm else 0.0
        print(wp.compare_measured(reqs, world, B, traces, lists, t_comm=t_comm, fmt=args.fmt), end="", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
