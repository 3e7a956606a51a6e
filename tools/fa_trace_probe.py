"""Timeline of CTA 0 of the fused attention forward (library built with
-DWP_FA_TRACE): per (event, warpgroup, step) SM clock, printed in time order."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_15762_b200 import _native  # noqa: E402

lib = _native.lib
lib.wp_debug_flash_fwd.argtypes = [C.c_int] * 5 + [C.c_void_p] * 3
lib.wp_debug_fa_trace.argtypes = [C.c_void_p, C.c_int]
NAMES = {1: "S_commit", 2: "PV_commit", 3: "sm_wait_S", 4: "sm_got_S", 5: "sm_wait_O", 6: "sm_got_O",
         7: "sm_P_ready", 8: "mma_enter_S", 9: "mma_enter_PV", 10: "mma_issue_S", 11: "mma_issue_PV"}
mbs, seq, heads, d = 8, 1024, 16, int(os.environ.get("D", "128"))
causal = int(sys.argv[1]) if len(sys.argv) > 1 else 0
h = heads * d
qkv = torch.randn(mbs * seq, 3 * h, device="cuda").bfloat16()
ctx = torch.empty(mbs * seq, h, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(mbs, heads, seq, device="cuda")
for _ in range(3):
    lib.wp_debug_flash_fwd(mbs, seq, heads, d, causal, qkv.data_ptr(), ctx.data_ptr(), lse.data_ptr())
buf = (C.c_ulonglong * 1024)()
lib.wp_debug_fa_trace(buf, 1024)
ev = []
for e in range(16):
    for x in range(2):
        for j in range(32):
            t = buf[(e * 2 + x) * 32 + j]
            if t:
                ev.append((t, e, x, j))
ev.sort()
t0 = ev[0][0]
for t, e, x, j in ev:
    print(f"{t - t0:8d} {'AB'[x]} j={j:2d} {NAMES.get(e, e)}")
