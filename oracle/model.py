"""CPU fp32/fp64 restatement of the stage compute -- TEST ORACLE ONLY.

The reference has no model ("no tensor shapes, no parameter
contents"), so model numerics are "parity unpinned" by the reference: this
file is the builder's restatement of the model the runtime implements
(paper_2308_15762_b200/csrc/runtime/model.cpp), in plain torch CPU autograd.
Only tests/ and bench.py's cpu_baseline leg use it.

What the pipelined step must equal (synchronous flush): the
sequential gradient-accumulation step over all B microbatches,
    loss = mean_b mean_tokens CE(model(tokens_b), labels_b),
whatever the schedule's per-device order (src/schedule.cpp) or the slice
placement (src/placement.cpp:52-68) -- only the float summation order
differs, which the tolerances absorb.
"""
import math

import torch


def param_specs(desc):
    """Ordered (name, shape, init_std, init_value): mirrors unit_params()."""
    h, f, V, s, L = desc.hidden, desc.ffn, desc.vocab, desc.seq, desc.layers
    std_w, std_out = 0.02, 0.02 / math.sqrt(2.0 * L)
    out = [("wte", (V, h), std_w, 0.0), ("wpe", (s, h), std_w, 0.0)]
    for l in range(L):
        p = f"h.{l}."
        out += [(p + "ln1.w", (h,), 0, 1.0), (p + "ln1.b", (h,), 0, 0.0),
                (p + "attn.qkv.w", (3 * h, h), std_w, 0.0), (p + "attn.qkv.b", (3 * h,), 0, 0.0),
                (p + "attn.proj.w", (h, h), std_out, 0.0), (p + "attn.proj.b", (h,), 0, 0.0),
                (p + "ln2.w", (h,), 0, 1.0), (p + "ln2.b", (h,), 0, 0.0),
                (p + "mlp.fc1.w", (f, h), std_w, 0.0), (p + "mlp.fc1.b", (f,), 0, 0.0),
                (p + "mlp.fc2.w", (h, f), std_out, 0.0), (p + "mlp.fc2.b", (h,), 0, 0.0)]
    out += [("lnf.w", (h,), 0, 1.0), ("lnf.b", (h,), 0, 0.0)]
    if not desc.tie_embeddings:
        out.append(("lm_head.w", (V, h), std_w, 0.0))
    return out


def init_params(desc, seed=1234, nonzero_vectors=True):
    """Seeded fp32 parameters (torch.Generator on CPU).  nonzero_vectors makes
    LN/bias vectors random too, so their gradients are exercised."""
    g = torch.Generator().manual_seed(seed)
    params = {}
    for name, shape, std, val in param_specs(desc):
        if std > 0:
            t = torch.randn(shape, generator=g, dtype=torch.float32) * std
        elif nonzero_vectors:
            t = torch.full(shape, val, dtype=torch.float32) + 0.1 * torch.randn(shape, generator=g)
        else:
            t = torch.full(shape, val, dtype=torch.float32)
        params[name] = t
    return params


def gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x * x * x)))


def gelu_grad(x):
    t = torch.tanh(0.7978845608028654 * (x + 0.044715 * x * x * x))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * x * x)


# --- bf16 rounding-point emulation ------------------------------------------
# The runtime's bf16 mode (csrc/runtime/executor.cpp unit_fwd / unit_bwd) keeps
# fp32 masters and accumulates every GEMM in fp32, but stores these tensors in
# bf16: the weight shadows the GEMMs read, every activation it stashes or
# hands to the next unit (residual stream x, LayerNorm outputs, qkv, ctx, the
# GELU pre-activation and output, logits), and every data gradient it
# materialises (dx, dLN, dqkv, dctx, dU, dlogits).  `emulate="bf16"` rounds
# at exactly those points (round-to-nearest-even, like __float2bfloat16_rn),
# in the oracle's own dtype otherwise, so the GPU step can be held to a
# tolerance set by accumulation order rather than by bf16 storage.

def _bf16(x):
    return x.to(torch.bfloat16).to(x.dtype)


class _RoundBoth(torch.autograd.Function):
    """A tensor stored in bf16 whose gradient is also stored in bf16."""

    @staticmethod
    def forward(ctx, x):
        return _bf16(x)

    @staticmethod
    def backward(ctx, g):
        return _bf16(g)


def _round_value(x):
    """A bf16 copy read by a GEMM (weight shadows): the gradient flows to the
    fp32 master unrounded (weight gradients accumulate in fp32)."""
    return x + (_bf16(x) - x).detach()


class _GeluStored(torch.autograd.Function):
    """FC1 epilogue (kEpiGelu, kernels/tc_common.cuh): stores u in bf16 and
    y = bf16(gelu(bf16(u))); FC2's data-gradient epilogue (kEpiDGelu) stores
    dU = bf16((dY W2) * gelu'(bf16 u))."""

    @staticmethod
    def forward(ctx, u):
        ur = _bf16(u)
        ctx.save_for_backward(ur)
        return _bf16(gelu(ur))

    @staticmethod
    def backward(ctx, g):
        (ur,) = ctx.saved_tensors
        return _bf16(g * gelu_grad(ur))


class _Rounding:
    def __init__(self, mode):
        self.on = mode == "bf16"

    def both(self, x):
        return _RoundBoth.apply(x) if self.on else x

    def w(self, x):
        return _round_value(x) if self.on else x

    def gelu(self, u):
        return _GeluStored.apply(u) if self.on else gelu(u)


def layernorm(x, w, b, eps=1e-5):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) / torch.sqrt(var + eps) * w + b


def attn_block(P, l, x, desc, R=_Rounding(None)):
    p = f"h.{l}."
    mbs, s, h = x.shape
    H, d = desc.heads, h // desc.heads
    a = R.both(layernorm(x, P[p + "ln1.w"], P[p + "ln1.b"]))
    qkv = R.both(a @ R.w(P[p + "attn.qkv.w"]).T + P[p + "attn.qkv.b"])
    q, k, v = qkv.split(h, dim=-1)
    q, k, v = (t.reshape(mbs, s, H, d).transpose(1, 2) for t in (q, k, v))
    sc = (q @ k.transpose(-1, -2)) / math.sqrt(d)
    if desc.causal:
        mask = torch.triu(torch.ones(s, s, dtype=torch.bool), diagonal=1)
        sc = sc.masked_fill(mask, float("-inf"))
    pr = torch.softmax(sc, dim=-1)
    ctx = R.both((pr @ v).transpose(1, 2).reshape(mbs, s, h))
    return R.both(x + ctx @ R.w(P[p + "attn.proj.w"]).T + P[p + "attn.proj.b"])


def mlp_block(P, l, x, R=_Rounding(None)):
    p = f"h.{l}."
    a = R.both(layernorm(x, P[p + "ln2.w"], P[p + "ln2.b"]))
    u = a @ R.w(P[p + "mlp.fc1.w"]).T + P[p + "mlp.fc1.b"]
    return R.both(x + R.gelu(u) @ R.w(P[p + "mlp.fc2.w"]).T + P[p + "mlp.fc2.b"])


def microbatch_loss(P, tokens, labels, desc, emulate=None):
    """Mean token cross-entropy of one microbatch; tokens/labels [mbs, seq].
    emulate="bf16": round at the runtime's bf16 storage points (see above)."""
    R = _Rounding(emulate)
    tokens = torch.as_tensor(tokens, dtype=torch.long)
    labels = torch.as_tensor(labels, dtype=torch.long)
    x = R.both(R.w(P["wte"])[tokens] + R.w(P["wpe"])[torch.arange(tokens.shape[1])])
    for l in range(desc.layers):
        x = attn_block(P, l, x, desc, R)
        x = mlp_block(P, l, x, R)
    hf = R.both(layernorm(x, P["lnf.w"], P["lnf.b"]))
    W = P["wte"] if desc.tie_embeddings else P["lm_head.w"]
    logits = R.both(hf @ R.w(W).T)
    return torch.nn.functional.cross_entropy(logits.reshape(-1, logits.shape[-1]), labels.reshape(-1))


def reference_step(params, tokens, labels, desc, dtype=torch.float64, emulate=None):
    """Sequential gradient accumulation over the B microbatches.
    Returns (loss, {name: grad}) in `dtype`.  emulate="bf16" rounds at the
    bf16 runtime's storage points (the loss scale 1/B is folded into the
    dlogits the runtime stores, as xent_fwd_bwd does)."""
    P = {k: v.detach().to(dtype).clone().requires_grad_(True) for k, v in params.items()}
    B = tokens.shape[0]
    total = None
    for b in range(B):
        lb = microbatch_loss(P, tokens[b], labels[b], desc, emulate) / B
        lb.backward()
        total = lb.detach() if total is None else total + lb.detach()
    return float(total), {k: v.grad.detach().clone() for k, v in P.items()}


def sgd_update(params, grads, lr, weight_decay=0.0):
    """Mirror of optim_k kind 0 (kernels/ops.cu)."""
    return {k: (p.double() - lr * (grads[k].double() + weight_decay * p.double())) for k, p in params.items()}


def adamw_update(params, grads, lr, beta1, beta2, eps, weight_decay, step=1):
    """One AdamW step from zero state (mirror of optim_k kind 1)."""
    out = {}
    bc1, bc2 = 1 - beta1 ** step, 1 - beta2 ** step
    for k, p in params.items():
        g = grads[k].double()
        m = (1 - beta1) * g
        v = (1 - beta2) * g * g
        p = p.double()
        out[k] = p - lr * ((m / bc1) / (torch.sqrt(v / bc2) + eps) + weight_decay * p)
    return out
