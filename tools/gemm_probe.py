"""One tcgen05 GEMM and one cuBLAS GEMM of the same shape (for ncu)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2308_15762_b200 import _native  # noqa: E402

lib = _native.lib
lib.wp_debug_gemm.restype = C.c_int
lib.wp_debug_gemm.argtypes = [C.c_int] * 6 + [C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_int64] * 2 + \
    [C.c_int, C.c_float, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
M, N, K = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 8192, 8192)))
gelu = len(sys.argv) > 4 and sys.argv[4] == "gelu"
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
aux = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if gelu else None
bias = torch.zeros(N, device="cuda") if gelu else None
lib.wp_last_error.restype = C.c_char_p
for _ in range(2):
    st = lib.wp_debug_gemm(M, N, K, 1, 1, 1, a.data_ptr(), K, 0, 0, 0, b.data_ptr(), K, 0, 0, 0, 3 if gelu else 0, 1.0,
                      c.data_ptr(), 1, N, 0, 0, bias.data_ptr() if gelu else None, None,
                      aux.data_ptr() if gelu else None)
    assert st == 0, lib.wp_last_error().decode()
    torch.matmul(a, b.t())
torch.cuda.synchronize()
