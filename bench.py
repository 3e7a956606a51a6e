"""Benchmark: Hanayo wave-pipeline training step on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl wavepipe|reference]

Workload (BASELINE.json configs[3]): GPT-1.3B-like (24 layers, hidden 2048,
16 heads, ffn 8192, seq 1024, vocab 50304, tied embeddings), bf16 tensor-core
compute with fp32 master weights and AdamW, Hanayo W=2 over P=N GPUs
(N=1: all S=4 slices resident on one GPU), B=8 microbatches of 16 sequences
(global batch 128 x 1024 tokens; --mbs 4 / 8 / 16 measured 100 / 111 / 118
samples/s on one B200: larger microbatches feed the GEMMs M = 16384 rows),
synthetic tokens (splitmix64), random-init weights.

One "step" = one full synchronous training iteration: every microbatch's
forward and backward through every slice, the flush, and the optimizer
update.  `value` is samples/s with inputs resident in HBM; `e2e` is the same
step through the public API with the token/label batch copied from pinned
host memory every step and the loss read back.  The per-step working set
(~35 GB of weights, optimizer state and activations) is far larger than the
126 MB L2, so no explicit flush is needed between steps.

Multi-GPU: one rank per GPU.  `--gpus N` (N > 1) outside torchrun re-launches
itself under `torch.distributed.run` with N ranks; under torchrun WORLD_SIZE
must equal --gpus.  Rank r = pipeline device r; the inter-stage transport is
the CUDA-IPC one (copy-engine pushes over NVLink into IPC-mapped landing
slots, stream-memory-op flags; no fallback: a failed peer probe stops the
run); fixed global batch (strong scaling); time = max over ranks.  The
measured bubble merges every rank's trace (each relative to its own step
start, taken right after a barrier).  WP_BENCH_SHARE_GPU=1 maps every rank to
cuda:0 (functional testing of the multi-process path on a 1-GPU box; not a
measurement).

The reference arm (`--impl reference`) never imports this repo's package: its
workload description, inputs (oracle/data.py) and CPU step (oracle/model.py)
are test infrastructure, so only the oracle runs in that process.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

GPT13B = dict(layers=24, hidden=2048, heads=16, ffn=8192, seq=1024, vocab=50304)
# BASELINE.json configs as presets (--model); the default is the headline one.
MODELS = {
    "gpt-1.3b-like": dict(GPT13B, causal=True),
    "gpt2-medium-like": dict(layers=24, hidden=1024, heads=16, ffn=4096, seq=1024, vocab=50304, causal=True),
    "bert-large-like": dict(layers=24, hidden=1024, heads=16, ffn=4096, seq=512, vocab=30528, causal=False),
    "tiny-gpt": dict(layers=4, hidden=256, heads=4, ffn=1024, seq=128, vocab=1024, causal=True),
}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f), "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def flops_per_sample(m):
    """3 x forward FLOPs: L*(2*(4h^2+2hf) + a*s*h) + 2hV per token."""
    a = 2 if m["causal"] else 4
    h, f, s = m["hidden"], m["ffn"], m["seq"]
    return 3.0 * s * (m["layers"] * (2 * (4 * h * h + 2 * h * f) + a * s * h) + 2 * h * m["vocab"])


class Workload:
    """The benched model's shape without the product library (the reference
    arm and the CPU baseline use only this and oracle/)."""

    def __init__(self, args):
        self.m = dict(MODELS[getattr(args, "model", "gpt-1.3b-like")])
        for k, v in self.m.items():
            setattr(self, k, v)
        self.micro_batch_size = args.mbs
        self.tie_embeddings = True

    def flops_per_sample(self):
        return flops_per_sample(self.m)


def model_desc(args):
    import paper_2308_15762_b200 as wp
    m = MODELS[getattr(args, "model", "gpt-1.3b-like")]
    return wp.ModelDesc(**m, micro_batch_size=args.mbs, tie_embeddings=True, dtype="bf16",
                        optimizer="adamw", lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.01, seed=1234)


def cpu_port_sample(desc, threads=None):
    """Time the oracle's torch-CPU fp32 train step on a bounded sample: one
    sequence through (embedding + 1 transformer layer + LM head) at the full
    hidden/ffn/seq/vocab, forward+backward; extrapolate to samples/s of the
    full model by FLOPs (work conservation, proj/tests/test_simulate.cpp:67-79)."""
    import torch
    from oracle import model as om
    from oracle.data import synthetic_batch
    threads = threads or os.cpu_count()
    torch.set_num_threads(threads)

    class D:
        pass

    d1 = D()
    for k in ("layers", "hidden", "heads", "ffn", "seq", "vocab", "micro_batch_size", "causal",
              "tie_embeddings"):
        setattr(d1, k, getattr(desc, k))
    d1.layers, d1.micro_batch_size = 1, 1
    params = om.init_params(d1, seed=1, nonzero_vectors=False)
    tok, lab = synthetic_batch(1, 1, d1.seq, d1.vocab)
    t0 = time.perf_counter()
    om.reference_step(params, tok, lab, d1, dtype=torch.float32)
    dt = time.perf_counter() - t0
    a = 2 if desc.causal else 4
    h, f, s = desc.hidden, desc.ffn, desc.seq
    reduced = 3.0 * s * ((2 * (4 * h * h + 2 * h * f) + a * s * h) + 2 * h * desc.vocab)
    rate = reduced / dt
    return rate / flops_per_sample(dict(layers=desc.layers, hidden=h, ffn=f, seq=s, vocab=desc.vocab,
                                        causal=desc.causal)), dt, threads


# Full-step CPU path when the whole step is small enough to time directly
# (C1 on the full action list; larger models extrapolate).
FULL_LIST_TFLOP = 2.0


def cpu_full_list_step(args, P, threads=None):
    """Time the oracle's torch-CPU fp32 interpreter of the whole Hanayo action
    list (the reference's generator restated in oracle/schedule.py, pinned to
    its goldens) over B microbatches; returns (samples/s, seconds, threads)."""
    import torch
    from oracle import model as om
    from oracle import pipeline as opl
    from oracle import schedule as osch
    from oracle.data import synthetic_batch
    threads = threads or os.cpu_count()
    torch.set_num_threads(threads)
    desc = Workload(args)
    cfg = osch.make_config(osch.HANAYO, P, args.microbatches, args.waves)
    acts, pl = osch.generate_schedule(cfg)
    placement = [[sl[0] for sl in row] for row in pl]
    params = {k: v.float() for k, v in om.init_params(desc, seed=1).items()}
    tokens, labels = synthetic_batch(args.microbatches, args.mbs, desc.seq, desc.vocab)
    t0 = time.perf_counter()
    opl.run_local(desc, params, acts, placement, args.microbatches, tokens, labels, dtype=torch.float32)
    dt = time.perf_counter() - t0
    return args.microbatches * args.mbs / dt, dt, threads


def ref_schedule_time(P, B, W):
    """The reference's own CPU path (oracle/_ref: its src/*.cpp, generate +
    simulate), single-threaded as the reference is."""
    drv = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    if not os.path.exists(drv):
        return None
    out = subprocess.run([drv, "time", "hanayo", str(P), str(B), str(W), "5"], capture_output=True, text=True)
    try:
        return json.loads(out.stdout)["best_ms"]
    except (ValueError, KeyError):
        return None


def run_reference(args, rank, world):
    """Reference arm: the reference's CPU implementation of the path, timed on
    this box's host cores (rank 0 only)."""
    if rank != 0:
        return
    desc = Workload(args)
    P = args.gpus
    full = desc.flops_per_sample() * args.microbatches * args.mbs <= FULL_LIST_TFLOP * 1e12
    sample_fn = (lambda: cpu_full_list_step(args, P)) if full else (lambda: cpu_port_sample(Workload(args)))
    for _ in range(args.warmup):
        sample_fn()
    vals, per = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, dt, cores = sample_fn()
        vals.append(v)
        per.append(dt)
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    ref_ms = ref_schedule_time(P, args.microbatches, args.waves)
    sched = (f"schedule generate+simulate by the reference's own code (oracle/_ref): "
             f"{ref_ms if ref_ms is not None else 'n/a'} ms")
    if full:
        sample = (f"the whole Hanayo P={P} W={args.waves} B={args.microbatches} action list of {args.model} "
                  f"(mbs {args.mbs}), fp32 torch CPU interpreter ({statistics.median(per):.2f} s per step); {sched}")
    else:
        sample = (f"1 sequence x (embedding + 1 of {desc.layers} layers + LM head) of {args.model}, fp32 torch CPU "
                  f"fwd+bwd ({statistics.median(per):.2f} s), extrapolated to the full model by FLOPs; {sched}")
    line = {
        "impl": "reference", "metric": "samples/sec (Hanayo W=2 train step)", "value": value,
        "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic tokens (splitmix64), random-init weights",
        "config": workload_config(args, P * args.replicas),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, world):
    D = getattr(args, "replicas", 1)
    P = world // D
    par = f"pp{P}" + (f"xdp{D}" if D > 1 else "")
    name = getattr(args, "model", "gpt-1.3b-like")
    m = MODELS[name]
    return {"workload": "%s train step, Hanayo W=%d over P=%d" % (name, args.waves, P)
            + (f", {D} data-parallel replicas" if D > 1 else ""),
            "model": name, "layers": m["layers"], "hidden": m["hidden"], "heads": m["heads"], "ffn": m["ffn"],
            "seq_len": m["seq"], "vocab": m["vocab"], "micro_batch_size": args.mbs, "microbatches": args.microbatches,
            "global_batch": args.mbs * args.microbatches * D, "schedule": f"hanayo P={P} W={args.waves} "
            f"B={args.microbatches}" + (f" D={D}" if D > 1 else ""), "parallelism": par, "optimizer": "adamw",
            "l2_flush": l2_note(m, P)}


def l2_note(m, P):
    """Per-GPU bytes one step must touch at least: the slice parameters as
    bf16 shadow + fp32 master, gradient and AdamW m, v (18 B per parameter)."""
    h, f, L = m["hidden"], m["ffn"], m["layers"]
    params = L * (4 * h * h + 2 * h * f + 9 * h + f) + m["vocab"] * h + m["seq"] * h
    ws = 18 * params / P
    if ws > 126e6:
        return "not needed: per-step working set >= %.1f GB per GPU (parameter state alone) >> 126 MB L2" % (ws / 1e9)
    return "working set (%.0f MB) fits in L2: functional preset, not a timing configuration" % (ws / 1e6)


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_command(n, argv):
    """torchrun command line running this script on n ranks of this node."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + list(argv)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="wavepipe", choices=["wavepipe", "reference"])
    ap.add_argument("--microbatches", type=int, default=8)
    ap.add_argument("--mbs", type=int, default=16)
    ap.add_argument("--model", default="gpt-1.3b-like", choices=sorted(MODELS),
                    help="BASELINE.json config preset (default: the headline GPT-1.3B-like)")
    ap.add_argument("--waves", type=int, default=2)
    ap.add_argument("--replicas", type=int, default=1,
                    help="data-parallel replicas D (world = P*D ranks; IPC transport, peer-memory grad all-reduce)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gemm-report", action="store_true", help="per-shape GEMM table on stderr")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "wavepipe":
        # One process per GPU: re-launch under torchrun with --gpus ranks.
        os.execv(sys.executable, spawn_command(args.gpus, sys.argv[1:]))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "wavepipe" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch N ranks for --gpus N")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2308_15762_b200 as wp
    from paper_2308_15762_b200.data import synthetic_batch

    share = os.environ.get("WP_BENCH_SHARE_GPU") == "1"
    dev = 0 if share else local_rank
    torch.cuda.set_device(dev)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    D = args.replicas
    if world % D:
        raise SystemExit("--replicas must divide the number of ranks")
    P = world // D
    replica = rank // P
    desc = model_desc(args)
    cfg = wp.make_config(wp.Scheme.Hanayo, P, args.microbatches, args.waves, D)
    sched = wp.generate_schedule(cfg)
    transport = "ipc"
    if world > 1:
        rt = wp.Runtime(desc, sched, transport=wp.TRANSPORT_IPC, device_ids=[dev], rank=rank)
        ok, why = rt.ipc_status()
        flag = torch.tensor([1 if ok else 0], device="cpu" if share else "cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            raise SystemExit(f"rank {rank}: CUDA-IPC peer probe failed on this box ({why or 'a peer failed'})")
    else:
        rt = wp.Runtime(desc, sched, device_ids=[dev])

    tok_np, lab_np = synthetic_batch(args.microbatches, args.mbs, desc.seq, desc.vocab, step=replica)
    tok_d = torch.from_numpy(tok_np).cuda()
    lab_d = torch.from_numpy(lab_np).cuda()
    tok_h = torch.from_numpy(tok_np).pin_memory()
    lab_h = torch.from_numpy(lab_np).pin_memory()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(steps, host):
        barrier()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        loss = None
        for _ in range(steps):
            loss = rt.train_step(tok_h, lab_h) if host else rt.train_step(tok_d, lab_d)
        en.record()
        barrier()
        sec = st.elapsed_time(en) / 1e3
        if world > 1:
            t = torch.tensor([sec], device="cpu" if share else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = float(t.item())
            lt = torch.tensor([loss], device="cpu" if share else "cuda")
            dist.all_reduce(lt)  # the loss lives on the rank holding the head slice
            loss = float(lt.item()) / D  # mean over replicas
        return sec, loss

    for _ in range(args.warmup):
        rt.train_step(tok_d, lab_d)

    # Device-resident timed region (value), with clocks sampled during it.
    launches0 = rt.launch_count()
    clocks = ClockSampler(dev)
    clocks.start()
    sec, loss = timed(args.steps, host=False)
    clk = clocks.stop()
    launches = rt.launch_count() - launches0

    # End-to-end through the public API from pinned host buffers.
    sec_e2e, _ = timed(args.steps, host=True)

    # Per-kernel-class device time (roofline / attention objects) from a
    # separate profiled pass: the per-launch events it records would
    # otherwise slow the timed region above.
    rt.set_profiling(True)
    prof_steps = max(2, args.steps // 2)
    sec_prof, _ = timed(prof_steps, host=False)
    g_launches, g_flops, g_sec = rt.gemm_stats()
    a_launches, a_flops, a_sec = rt.attn_stats()
    hbm_raw = rt.hbm_stats()
    if args.gemm_report and rank == 0:
        print(rt.gemm_report(), file=sys.stderr, flush=True)
    rt.set_profiling(False)
    g_launches //= prof_steps
    a_launches //= prof_steps

    # One traced step: measured vs simulated bubble.  Each rank traces its
    # own pipeline device relative to its step start (right after a
    # barrier); rank 0 merges them into one trace (wp_trace_build).
    rt.set_tracing(True)
    barrier()
    rt.train_step(tok_d, lab_d)
    rt.set_tracing(False)
    tr = rt.trace()
    if world > 1:
        # replica 0's pipeline devices make up the measured trace of the list;
        # each rank's trace starts at its own step begin, so put them on one
        # device clock (%globaltimer at each rank's step begin) before merging
        pipe = rank % P
        mine = (tr.intervals[pipe], [e for e in tr.comm_events if e.src_device == pipe], rt.step_clock_ns())
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        t0 = min(p[2] for p in parts[:P])
        off = [(p[2] - t0) * 1e-9 for p in parts[:P]]
        tr = wp.build_trace([[iv._replace(start=iv.start + off[d], end=iv.end + off[d]) for iv in parts[d][0]]
                             for d in range(P)],
                            [e._replace(post_time=e.post_time + off[d], arrival_time=e.arrival_time + off[d])
                             for d in range(P) for e in parts[d][1]])
    measured_bubble = wp.bubble_ratio(tr)
    pool_b, landing_b = rt.memory()
    mem = [None] * world
    if world > 1:
        dist.all_gather_object(mem, (pool_b, landing_b))
    else:
        mem = [(pool_b, landing_b)]
    msg_bytes = desc.tokens_per_microbatch * desc.hidden * 2
    copies = [e.arrival_time - e.post_time for e in tr.comm_events if e.arrival_time > e.post_time]
    p2p = {"messages": len(tr.comm_events), "bytes_per_message": msg_bytes,
           "mean_copy_us": 1e6 * statistics.mean(copies) if copies else None,
           "mean_copy_gbs": msg_bytes / statistics.mean(copies) / 1e9 if copies else None,
           "transport": transport if world > 1 else "none (P=1)"}
    fwd = [iv.end - iv.start for dev in tr.intervals for iv in dev if iv.kind == wp.ActionKind.Forward]
    bwd = [iv.end - iv.start for dev in tr.intervals for iv in dev if iv.kind == wp.ActionKind.Backward]
    tf, tb = statistics.mean(fwd) * 2 * args.waves, statistics.mean(bwd) * 2 * args.waves
    sim = wp.simulate(sched, wp.CostModel(tf, tb, 0.0))
    sim_bubble = wp.bubble_ratio(sim)
    eq1 = wp.analytic_bubble_hanayo_d(P, args.waves, tf, tb, 0.0) if P >= 2 else None

    if rank != 0:
        dist.barrier()  # peers' IPC mappings stay valid until every rank is done
        rt.close()
        dist.destroy_process_group()
        return
    samples = args.microbatches * args.mbs * args.steps * D
    value = samples / sec
    peaks, peaks_kind = load_peaks()
    peak_tc = peaks.get("bf16_tflops_sustained", PEAKS_FALLBACK["bf16_tflops_sustained"])
    achieved = g_flops / g_sec / 1e12 if g_sec > 0 else None
    # DRAM bytes per launch (ncu --set full, tools/traffic.py) of the dominant
    # GEMM (FC1 forward, the most expensive shape) and of the attention
    # backward, next to their algorithmic bytes -- used only when captured at
    # this run's shapes.
    traffic_all = {}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic_all = json.load(f)
    except (OSError, ValueError):
        pass
    T = args.mbs * desc.seq

    def traffic_for(key, shape):
        t = traffic_all.get(key)
        if not t or list(t.get("shape", [])) != list(shape):
            return None
        return {k: t.get(k) for k in ("shape", "bytes_per_launch", "algorithmic_bytes", "ratio", "source")}

    fc1 = traffic_for("gemm_fc1", [T, desc.ffn, desc.hidden])
    attn_bwd_traffic = traffic_for("flash_bwd", [args.mbs, desc.heads, desc.seq, desc.hidden // desc.heads,
                                                 int(desc.causal)])
    hbm_peak = peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])
    hbm = {"peak_gbs": hbm_peak, "peak_kind": f"{peaks_kind} STREAM-style copy", "kernels": {},
           "share_of_step": sum(v[2] for v in hbm_raw.values()) / sec_prof if sec_prof > 0 else None,
           "bytes": "algorithmic (reads + writes of the tensors each launch must touch), per launch"}
    for name, (n, b, t) in sorted(hbm_raw.items()):
        if n == 0 or t <= 0:
            continue
        hbm["kernels"][name] = {"launches_per_step": n / prof_steps, "bytes_per_launch": b / n,
                                "us_per_launch": 1e6 * t / n, "achieved_gbs": b / t / 1e9,
                                "frac": b / t / 1e9 / hbm_peak}
    flops_step = flops_per_sample(MODELS[args.model]) * args.microbatches * args.mbs * D
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        if flops_step <= FULL_LIST_TFLOP * 1e12:
            v, dt, cores = cpu_full_list_step(args, 1)
            smp = (f"the whole Hanayo P=1 W={args.waves} B={args.microbatches} action list, fp32 torch CPU "
                   f"interpreter ({dt:.2f} s per step)")
        else:
            v, dt, cores = cpu_port_sample(desc)
            smp = (f"1 sequence x (embedding + 1 of {desc.layers} layers + LM head), fp32 torch CPU fwd+bwd "
                   f"({dt:.2f} s), extrapolated to the {desc.layers}-layer model by FLOPs")
        cpu = {"value": v, "unit": "samples/s", "cores": cores, "kind": "port", "sample": smp}
    line = {
        "metric": "samples/sec (Hanayo W=2 train step)", "value": value, "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic tokens (splitmix64), random-init weights",
        "config": workload_config(args, world),
        "tc_peak_frac": flops_step * args.steps / sec / world / (peak_tc * 1e12),
        "bubble": {"measured": measured_bubble, "simulated_at_measured_costs": sim_bubble, "eq1": eq1,
                   "clock": "per-rank traces aligned on %globaltimer at step begin" if world > 1 else "one device",
                   "t_forward_s": tf, "t_backward_s": tb},
        "p2p": p2p,
        "memory": {"stash_pool_gb_max": max(m[0] for m in mem) / 1e9,
                   "landing_gb_max": max(m[1] for m in mem) / 1e9,
                   "reference_peak_activation_units": [str(u) for u in wp.memory_profile(sim, sched)[1]]},
        "roofline": {"bound": "tensor", "kernel": "gemm_tc (tcgen05, all GEMM launches of the step)",
                     "achieved": achieved, "peak": peak_tc, "unit": "TFLOP/s",
                     "frac": achieved / peak_tc if achieved else None,
                     "traffic": fc1["bytes_per_launch"] if fc1 else None, "traffic_launch": fc1,
                     "peak_kind": f"{peaks_kind} bf16 sustained (kernel timed inside a long step)",
                     "gemm_launches": g_launches, "gemm_share_of_step": g_sec / sec_prof},
        "attention": {"kernel": "flash_fwd_kernel / flash_bwd_kernel (tcgen05)", "launches": a_launches,
                      "achieved_tflops": a_flops / a_sec / 1e12 if a_sec > 0 else None,
                      "frac_of_peak": a_flops / a_sec / 1e12 / peak_tc if a_sec > 0 else None,
                      "share_of_step": a_sec / sec_prof if sec_prof > 0 else None,
                      "traffic_bwd_launch": attn_bwd_traffic},
        "hbm": hbm,
        "cpu_baseline": cpu,
        "e2e": {"value": samples / sec_e2e, "unit": "samples/s",
                "h2d_bytes_per_step": int(tok_h.numel() * 4 + lab_h.numel() * 4), "d2h_bytes_per_step": 4},
        "gpu_launches": launches,
        "clocks": clk,
        "loss": loss,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
    rt.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
