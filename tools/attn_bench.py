"""Time the fused attention kernels at the bench shape (GPT-1.3B, mbs=8):
CUDA events around N back-to-back launches; algorithmic FLOPs (causal half)
fwd = 4*mbs*heads*seq^2*d/2, bwd = 2.5x fwd."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_15762_b200 import _native  # noqa: E402

lib = _native.lib
lib.wp_debug_flash_fwd.argtypes = [C.c_int] * 5 + [C.c_void_p] * 3
lib.wp_debug_flash_bwd.argtypes = [C.c_int] * 5 + [C.c_void_p] * 7


def main(mbs=8, seq=1024, heads=16, d=128, causal=1, n=20):
    h = heads * d
    qkv = torch.randn(mbs * seq, 3 * h, device="cuda").bfloat16()
    ctx = torch.empty(mbs * seq, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(mbs, heads, seq, device="cuda")
    dout = torch.randn(mbs * seq, h, device="cuda").bfloat16()
    delta = torch.empty(mbs, heads, seq, device="cuda")
    dq = torch.empty(mbs * seq, h, device="cuda")
    dqkv = torch.empty(mbs * seq, 3 * h, device="cuda", dtype=torch.bfloat16)
    fwd = lambda: lib.wp_debug_flash_fwd(mbs, seq, heads, d, causal, qkv.data_ptr(), ctx.data_ptr(), lse.data_ptr())
    bwd = lambda: lib.wp_debug_flash_bwd(mbs, seq, heads, d, causal, qkv.data_ptr(), ctx.data_ptr(), dout.data_ptr(),
                                         lse.data_ptr(), delta.data_ptr(), dq.data_ptr(), dqkv.data_ptr())
    flops = 4.0 * mbs * heads * seq * seq * d / (2 if causal else 1)
    for name, f, fl in (("fwd", fwd, flops), ("bwd", bwd, 2.5 * flops)):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(n):
            f()  # each call synchronises (debug entry); times include that
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / n
        print(f"{name}: {1e3 * ms:8.1f} us  {fl / ms / 1e9:7.1f} TFLOP/s  (mbs={mbs} seq={seq} heads={heads} d={d} "
              f"causal={causal})", flush=True)


if __name__ == "__main__":
    main()
    main(causal=0)
