"""Microbenchmark of the tcgen05 GEMM against torch.matmul (cuBLAS) on the
GPT-1.3B slice shapes (T = 4096 tokens).  Prints one JSON line per shape."""
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


def bench(M, N, K, a_mn=False, b_mn=False, iters=20):
    a = torch.randn((K, M) if a_mn else (M, K), device="cuda", dtype=torch.bfloat16)
    b = torch.randn((K, N) if b_mn else (N, K), device="cuda", dtype=torch.bfloat16)
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    args = (M, N, K, 1, 1, 1, a.data_ptr(), M if a_mn else K, int(a_mn), 0, 0,
            b.data_ptr(), N if b_mn else K, int(b_mn), 0, 0, 0, 1.0, c.data_ptr(), 1, N, 0, 0, None, None, None)
    assert lib.wp_debug_gemm(*args) == 0, lib.wp_last_error()
    # back-to-back asynchronous launches on the default stream, like cuBLAS below
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    st.record()
    for _ in range(iters):
        lib.wp_debug_gemm_async(*args)
    en.record()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en) / iters
    at = a.t() if a_mn else a
    bt = b if b_mn else b.t()
    for _ in range(3):
        torch.matmul(at, bt)
    torch.cuda.synchronize()
    st.record()
    for _ in range(iters):
        torch.matmul(at, bt)
    en.record()
    torch.cuda.synchronize()
    ms_ref = st.elapsed_time(en) / iters
    fl = 2.0 * M * N * K
    return {"M": M, "N": N, "K": K, "a_mn": a_mn, "b_mn": b_mn, "ms": ms, "tflops": fl / ms / 1e9,
            "cublas_ms": ms_ref, "cublas_tflops": fl / ms_ref / 1e9}


if __name__ == "__main__":
    T, h, f = 4096, 2048, 8192
    shapes = [(T, 3 * h, h), (T, h, h), (T, f, h), (T, h, f),          # fwd
              (T, h, 3 * h, False, True), (T, h, f, False, True),     # dgrad
              (3 * h, h, T, True, True), (f, h, T, True, True),       # wgrad
              (8192, 8192, 8192)]
    for s in shapes:
        print(json.dumps(bench(*s)), flush=True)
