"""tcgen05 GEMM epilogue modes at the slice shapes (M = mbs*seq = 16384):
store / residual / GELU / dGELU, back-to-back launches timed with CUDA
events.  Prints one JSON line per (shape, mode)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2308_15762_b200 import _native  # noqa: E402

lib = _native.lib
for _f in (lib.wp_debug_gemm, lib.wp_debug_gemm_async):
    _f.restype = C.c_int
    _f.argtypes = [C.c_int] * 6 + [C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_int64] * 2 + \
        [C.c_int, C.c_float, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
         C.c_void_p]
lib.wp_last_error.restype = C.c_char_p
NAMES = {0: "store", 2: "residual", 3: "gelu", 4: "dgelu"}


def bench(M, N, K, mode, b_mn=False, iters=20):
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn((K, N) if b_mn else (N, K), device="cuda", dtype=torch.bfloat16)
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    bias = torch.zeros(N, device="cuda")
    x = torch.randn(M, N, device="cuda", dtype=torch.bfloat16)
    args = (M, N, K, 1, 1, 1, a.data_ptr(), K, 0, 0, 0, b.data_ptr(), N if b_mn else K, int(b_mn), 0, 0, mode, 1.0,
            c.data_ptr(), 1, N, 0, 0, bias.data_ptr() if mode in (2, 3) else None,
            x.data_ptr() if mode == 2 else None, x.data_ptr() if mode in (3, 4) else None)
    assert lib.wp_debug_gemm(*args) == 0, lib.wp_last_error()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    st.record()
    for _ in range(iters):
        lib.wp_debug_gemm_async(*args)
    en.record()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en) / iters
    return {"M": M, "N": N, "K": K, "mode": NAMES[mode], "us": 1e3 * ms, "tflops": 2.0 * M * N * K / ms / 1e9}


if __name__ == "__main__":
    T = 16384
    for h, f in ((2048, 8192), (1024, 4096)):
        for (N, K, b_mn), modes in (((f, h, False), (0, 3)), ((f, h, True), (0, 4)), ((h, h, False), (0, 2)),
                                    ((h, f, False), (0, 2))):
            for m in modes:
                print(json.dumps(bench(T, N, K, m, b_mn)), flush=True)
