"""Per-parameter gradient error of the bf16 runtime vs the fp64 oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2308_15762_b200 as wp  # noqa: E402
from oracle import model as om  # noqa: E402
from paper_2308_15762_b200.data import synthetic_batch  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dtype = sys.argv[3] if len(sys.argv) > 3 else "bf16"
desc = wp.ModelDesc(layers=2, hidden=256, heads=4, ffn=1024, seq=128, vocab=1024, micro_batch_size=2, dtype=dtype)
sched = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, P, 4, W))
rt = wp.Runtime(desc, sched, device_ids=[0] * P)
params = om.init_params(desc, seed=7)
for n, t in params.items():
    rt.set_param(n, t.numpy())
rt.set_update(False)
tok, lab = synthetic_batch(4, 2, desc.seq, desc.vocab)
loss = rt.train_step(tok, lab)
ref_loss, g = om.reference_step(params, tok, lab, desc)
print("loss", loss, ref_loss)
for n, r in g.items():
    got = rt.get_grad(n, r.numel()).astype(np.float64)
    want = r.numpy().ravel()
    print(f"{n:24s} {np.linalg.norm(got - want) / np.linalg.norm(want):.3e}  |g|={np.linalg.norm(want):.3e}")
