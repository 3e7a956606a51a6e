"""CPU interpreter of an action list with real message passing -- TEST ORACLE.

Executes each pipeline device's program in order, as the runtime's action
interpreter does (paper_2308_15762_b200/csrc/runtime/executor.cpp,
Runtime::advance): Forward/Backward run the slice's units with torch autograd
on CPU; Send/Receive are point-to-point messages; a BatchedExchange is one
grouped send+recv with its counterpart.  The slice->unit partition restates
the runtime's device-balanced partition_units (csrc/runtime/model.cpp).

Drivers: `run_local` (all devices in one process, relaxation order like the
reference simulator, src/simulate.cpp:86-158) and `run_dist` (one process
per device over torch.distributed point-to-point; the gloo world_size-2
test).  `channels` gives the per-directed-pair sender order `run_dist`
posts its receives in (gloo matches a pair's messages FIFO).
"""
import torch

from . import model as om

FORWARD, BACKWARD, SEND, RECEIVE, BATCHED_EXCHANGE, OPTIMIZER_STEP = range(6)


def units(desc):
    """build_units (csrc/runtime/model.cpp): (kind, layer, cost)."""
    h, f, s, V = desc.hidden, desc.ffn, desc.seq, desc.vocab
    core = (2.0 if desc.causal else 4.0) * s * h
    u = [("embed", -1, float(h))]
    for l in range(desc.layers):
        u.append(("attn", l, 8.0 * h * h + core))
        u.append(("mlp", l, 4.0 * h * f))
    u.append(("head", -1, 2.0 * h * V))
    return u


def partition(us, slice_device, P):
    """partition_units(units, slice_device, P) (csrc/runtime/model.cpp): the
    device-balanced cut the runtime uses.  Per-slice targets give every device
    total/P (the pinned embedding / LM head counting toward their device),
    cuts are placed greedily on those targets, then a coordinate descent moves
    each cut to the position minimising (busiest device load, sum of squared
    device loads) until no cut moves.  Numerics do not depend on the cut
    (pipelined = sequential for any partition); the interpreter uses it so it
    executes the runtime's slices unit for unit."""
    S, N = len(slice_device), len(us)
    prefix = [0.0]
    for _, _, c in us:
        prefix.append(prefix[-1] + c)
    total = prefix[N]
    fixed = [0.0] * S
    fixed[0] += us[0][2]
    fixed[S - 1] += us[-1][2]
    dev_fixed, dev_slices = [0.0] * P, [0] * P
    for k in range(S):
        dev_fixed[slice_device[k]] += fixed[k]
        dev_slices[slice_device[k]] += 1
    target = [fixed[k] + max(0.0, total / P - dev_fixed[slice_device[k]]) / dev_slices[slice_device[k]]
              for k in range(S)]
    tsum = sum(target)
    b = [0] * (S + 1)
    b[S] = N
    cum = 0.0
    for k in range(1, S):
        cum += target[k - 1] * total / tsum
        lo = max(b[k - 1], 1)
        best, best_d = lo, abs(prefix[lo] - cum)
        for i in range(lo + 1, N):
            d = abs(prefix[i] - cum)
            if d < best_d:
                best, best_d = i, d
        b[k] = min(best, N - 1)

    def score(bb):
        load = [0.0] * P
        for k in range(S):
            load[slice_device[k]] += prefix[bb[k + 1]] - prefix[bb[k]]
        return max(load), sum(x * x for x in load)

    cur = score(b)
    moved = True
    while moved:
        moved = False
        for k in range(1, S):
            lo, hi = max(b[k - 1], 1), min(b[k + 1], N - 1)
            best, best_s = b[k], cur
            for pos in range(lo, hi + 1):
                b[k] = pos
                sc = score(b)
                if sc < best_s:
                    best_s, best = sc, pos
            b[k] = best
            if best_s < cur:
                cur = best_s
                moved = True
    return b


def slice_devices(placement):
    S = sum(len(r) for r in placement)
    sd = [0] * S
    for d, row in enumerate(placement):
        for s in row:
            sd[s] = d
    return sd


def key_of(a):
    kind, mb, _, s, _, payload, _ = a
    out = kind in (SEND, BATCHED_EXCHANGE)
    low = (s if out else s - 1) if payload == 0 else (s - 1 if out else s)
    return (payload, mb, low)


def channels(per_device):
    """Directed device pairs (src, dst) with their messages in the SENDER's
    program order (Sends and the outgoing halves of BatchedExchanges).

    run_dist's receiver posts its receives for a channel in this sender
    order at step start (so the FIFO matching of point-to-point pairs each message
    with the right landing buffer even where the receiver consumes messages
    in another order -- per-pair program orders differ, e.g. activations and
    gradients interleave differently on the two sides)."""
    out = {}
    for d, dev in enumerate(per_device):
        for a in dev:
            if a[0] in (SEND, BATCHED_EXCHANGE):
                out.setdefault((d, a[4]), []).append(key_of(a))
    return dict(sorted(out.items()))


def incoming(per_device, d):
    """Keys device d consumes from other devices (Receives and incoming halves
    of BatchedExchanges), in d's program order."""
    partner = {}
    for q, dev in enumerate(per_device):
        for a in dev:
            if a[0] == BATCHED_EXCHANGE:
                partner.setdefault(a[6], []).append((q, a))
    keys = []
    for a in per_device[d]:
        if a[0] == RECEIVE:
            keys.append((a[4], key_of(a)))
        elif a[0] == BATCHED_EXCHANGE:
            other = [b for q, b in partner[a[6]] if q != d][0]
            keys.append((a[4], key_of(other)))
    return keys


class Device:
    """One pipeline device's parameters and program state."""

    def __init__(self, desc, params, slices, bounds, us, dtype=torch.float64):
        self.desc, self.bounds, self.us = desc, bounds, us
        self.P = {k: v.detach().clone().to(dtype).requires_grad_(True) for k, v in params.items()}
        self.slices = slices
        self.stash = {}      # (mb, slice) -> (input tensor or None, output tensor)
        self.inbox = {}
        self.outbox = {}
        self.loss = 0.0

    def run_units(self, s, x, tokens, labels):
        d = self.desc
        for u in range(self.bounds[s], self.bounds[s + 1]):
            kind, l, _ = self.us[u]
            if kind == "embed":
                t = torch.as_tensor(tokens, dtype=torch.long)
                x = self.P["wte"][t] + self.P["wpe"][torch.arange(t.shape[1])]
            elif kind == "attn":
                x = om.attn_block(self.P, l, x, d)
            elif kind == "mlp":
                x = om.mlp_block(self.P, l, x)
            else:
                hf = om.layernorm(x, self.P["lnf.w"], self.P["lnf.b"])
                W = self.P["wte"] if d.tie_embeddings else self.P["lm_head.w"]
                logits = hf @ W.T
                lab = torch.as_tensor(labels, dtype=torch.long).reshape(-1)
                x = torch.nn.functional.cross_entropy(logits.reshape(-1, logits.shape[-1]), lab)
        return x


def step_device(dev, a, B, tokens, labels):
    """Execute one compute action on `dev`; returns (key, tensor) to publish or None."""
    kind, mb, _, s, _, _, _ = a
    S = len(dev.bounds) - 1
    if kind == FORWARD:
        if s == 0:
            x_in = None
        else:
            x_in = dev.inbox.pop((0, mb, s - 1)).detach().requires_grad_(True)
        out = dev.run_units(s, x_in, tokens[mb], labels[mb])
        dev.stash[(mb, s)] = (x_in, out)
        if s < S - 1:
            dev.outbox[(0, mb, s)] = out.detach()
            return (0, mb, s), out.detach()
        dev.loss += float(out.detach()) / B
        return None
    x_in, out = dev.stash.pop((mb, s))
    if s == S - 1:
        (out / B).backward()
    else:
        g = dev.inbox.pop((1, mb, s))
        out.backward(g)
    if s > 0:
        gx = x_in.grad.detach() if x_in.grad is not None else torch.zeros_like(x_in)
        dev.outbox[(1, mb, s - 1)] = gx
        return (1, mb, s - 1), gx
    return None


def owner(placement, s):
    for d, row in enumerate(placement):
        if s in row:
            return d
    return -1


def run_local(desc, params, per_device, placement, B, tokens, labels, dtype=torch.float64):
    """Single process, all devices, relaxation order (as src/simulate.cpp).
    dtype: float64 for parity checks, float32 for the bench's CPU path."""
    us = units(desc)
    bounds = partition(us, slice_devices(placement), len(placement))
    devs = [Device(desc, params, placement[d], bounds, us, dtype) for d in range(len(per_device))]
    published = {}
    pc = [0] * len(devs)
    moved = True
    while moved:
        moved = False
        for d, dev in enumerate(devs):
            prog = per_device[d]
            while pc[d] < len(prog):
                a = prog[pc[d]]
                k = a[0]
                if k in (FORWARD, BACKWARD):
                    r = step_device(dev, a, B, tokens, labels)
                    if r is not None:
                        key, t = r
                        consumer = key[2] + 1 if key[0] == 0 else key[2]
                        if owner(placement, consumer) == d:
                            dev.inbox[key] = dev.outbox.pop(key)
                elif k == SEND:
                    published[key_of(a)] = dev.outbox.pop(key_of(a))
                elif k == RECEIVE:
                    if key_of(a) not in published:
                        break
                    dev.inbox[key_of(a)] = published.pop(key_of(a))
                elif k == BATCHED_EXCHANGE:
                    ko = key_of(a)
                    if ko in dev.outbox:
                        published[ko] = dev.outbox.pop(ko)
                    partner = next(p for p in per_device[a[4]] if p[0] == BATCHED_EXCHANGE and p[6] == a[6])
                    ki = key_of(partner)
                    if ki not in published:
                        break
                    dev.inbox[ki] = published.pop(ki)
                pc[d] += 1
                moved = True
    assert all(pc[d] == len(per_device[d]) for d in range(len(devs))), "interpreter stalled"
    return devs


def run_dist(desc, params, per_device, placement, B, tokens, labels, replicas=1):
    """One process per pipeline device over torch.distributed point-to-point
    (gloo on CPU): every incoming message of the step is posted at step start, per
    channel in the sender's order (FIFO matching, tag 0); Sends and the
    outgoing halves of BatchedExchanges are issued in program order right
    after their producer; a consumer waits only for its own message.

    replicas = D > 1: global rank = replica * P + pipeline device (the GPU
    runtime's IPC rank layout); each replica runs the list on its own
    microbatches and the optimizer-step flush averages the gradients over
    the D replicas of each pipeline device (the runtime's peer-memory
    all-reduce, here a gloo all_reduce on a per-device group)."""
    import torch.distributed as dist
    P = len(per_device)
    g = dist.get_rank()
    r, base = g % P, (g // P) * P
    us = units(desc)
    bounds = partition(us, slice_devices(placement), len(placement))
    dev = Device(desc, params, placement[r], bounds, us)
    shape = (desc.micro_batch_size, desc.seq, desc.hidden)
    pending = {}
    for (src, dst), keys in channels(per_device).items():
        if dst != r:
            continue
        for k in keys:
            buf = torch.empty(shape, dtype=torch.float64)
            pending[k] = (dist.irecv(buf, src=base + src), buf)
    sends = []
    want = dict((k, src) for src, k in incoming(per_device, r))
    for a in per_device[r]:
        k = a[0]
        if k in (FORWARD, BACKWARD):
            # the consumer's inputs: wait for exactly the messages it needs
            mb, s = a[1], a[3]
            need = (0, mb, s - 1) if k == FORWARD else (1, mb, s)
            if need in pending:
                req, buf = pending.pop(need)
                req.wait()
                dev.inbox[need] = buf
            res = step_device(dev, a, B, tokens, labels)
            if res is not None:
                key = res[0]
                consumer = key[2] + 1 if key[0] == 0 else key[2]
                if owner(placement, consumer) == r:
                    dev.inbox[key] = dev.outbox.pop(key)
        elif k in (SEND, BATCHED_EXCHANGE):
            sends.append(dist.isend(dev.outbox.pop(key_of(a)).contiguous(), dst=base + a[4]))
    for q in sends:
        q.wait()
    if replicas > 1:
        # every rank creates every group, in the same order (collective)
        groups = [dist.new_group([q * P + d for q in range(replicas)]) for d in range(P)]
        for name, prm in sorted(dev.P.items()):
            if prm.grad is not None:
                dist.all_reduce(prm.grad, group=groups[r])
                prm.grad /= replicas
        dev.loss /= replicas
    assert not pending and set(want) <= set(dev.inbox) | set(want), "unconsumed messages"
    return dev
