"""Determinism probes: the same GEMM / train step twice must agree."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_15762_b200 as wp  # noqa: E402
from paper_2308_15762_b200 import _native  # noqa: E402
from paper_2308_15762_b200.data import synthetic_batch  # noqa: E402
from oracle import model as om  # noqa: E402

lib = _native.lib
lib.wp_debug_gemm.restype = C.c_int
lib.wp_debug_gemm.argtypes = [C.c_int] * 6 + [C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_int64] * 2 + \
    [C.c_int, C.c_float, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]


def gemm(M, N, K, a_mn, b_mn, mode=0):
    torch.manual_seed(0)
    a = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
    b = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
    outs = []
    for _ in range(4):
        c = torch.zeros(M, N, device="cuda")
        assert lib.wp_debug_gemm(M, N, K, 1, 1, 1, a.data_ptr(), M if a_mn else K, int(a_mn), 0, 0,
                                 b.data_ptr(), N if b_mn else K, int(b_mn), 0, 0, mode, 1.0, c.data_ptr(), 0, N, 0,
                                 0, None, None, None) == 0
        outs.append(c)
    ref = (a.float().t() if a_mn else a.float()) @ (b.float() if b_mn else b.float().t())
    same = all(torch.equal(outs[0], o) for o in outs[1:])
    err = ((outs[0] - ref).norm() / ref.norm()).item()
    print(f"gemm {M}x{N}x{K} a_mn={a_mn} b_mn={b_mn}: deterministic={same} relerr={err:.2e}")


for M, N, K in [(256, 256, 1024), (1024, 256, 256), (256, 1024, 256), (256, 768, 256), (768, 256, 256),
                (2048, 2048, 2048)]:
    for a_mn, b_mn in [(False, False), (False, True), (True, True)]:
        gemm(M, N, K, a_mn, b_mn)

desc = wp.ModelDesc(layers=1, hidden=256, heads=4, ffn=1024, seq=128, vocab=1024, micro_batch_size=2, dtype="bf16")
sched = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, 1, 2, 1))
rt = wp.Runtime(desc, sched, device_ids=[0])
params = om.init_params(desc, seed=7)
for n, t in params.items():
    rt.set_param(n, t.numpy())
rt.set_update(False)
tok, lab = synthetic_batch(2, 2, desc.seq, desc.vocab)
losses, grads = [], []
for _ in range(3):
    losses.append(rt.train_step(tok, lab))
    grads.append(rt.get_grad("lnf.b", 256).copy())
print("losses", losses)
print("lnf.b grad diffs", [float(np.abs(g - grads[0]).max()) for g in grads])
