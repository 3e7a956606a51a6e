"""GEMM kernels vs a torch fp32 reference of the same contraction (GPU).

Covers every operand-majorness combination the pipeline uses (X@W^T, dY@W,
dY^T@X, attention's Q@K^T / P@V / P^T@dO), two-level batching, M/N/K tails
and each fused epilogue, for both the tcgen05 bf16 kernel and the fp32 SIMT
parity kernel.
"""
import ctypes as C

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2308_15762_b200 import _native  # noqa: E402

lib = _native.lib
lib.wp_debug_gemm.restype = C.c_int
lib.wp_debug_gemm.argtypes = [C.c_int] * 6 + [C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_int64] * 2 + \
    [C.c_int, C.c_float, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
     C.c_void_p]

EPI_STORE, EPI_ACCUM, EPI_RESID, EPI_GELU, EPI_DGELU = range(5)


def gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def gelu_grad(x):
    t = torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * x * x)


def make_operand(rows, k, mn_major, dtype, batch=1):
    """Logical [batch, rows, k] operand stored row-major as [.., rows, k] (K-major)
    or [.., k, rows] (MN-major)."""
    if mn_major:
        store = torch.randn(batch, k, rows, device="cuda").to(dtype)
        logical = store.float().transpose(1, 2)
        ld = rows
    else:
        store = torch.randn(batch, rows, k, device="cuda").to(dtype)
        logical = store.float()
        ld = k
    return store, logical, ld


def run(M, N, K, a_mn, b_mn, dtype, mode=EPI_STORE, batch=1, bias=False, c_dtype=None, alpha=1.0):
    c_dtype = c_dtype or dtype
    in_code = 1 if dtype == torch.bfloat16 else 0
    c_code = 1 if c_dtype == torch.bfloat16 else 0
    a, al, lda = make_operand(M, K, a_mn, dtype, batch)
    b, bl, ldb = make_operand(N, K, b_mn, dtype, batch)
    acc = torch.bmm(al, bl.transpose(1, 2)) * alpha
    bias_t = torch.randn(N, device="cuda") if bias else None
    if bias_t is not None:
        acc = acc + bias_t
    c = torch.randn(batch, M, N, device="cuda").to(c_dtype)
    resid = torch.randn(batch, M, N, device="cuda").to(c_dtype) if mode == EPI_RESID else None
    aux = torch.randn(batch, M, N, device="cuda").to(c_dtype) if mode in (EPI_GELU, EPI_DGELU) else None
    c0 = c.float().clone()
    aux0 = aux.float().clone() if aux is not None else None
    st = lib.wp_debug_gemm(M, N, K, batch, 1, in_code,
                           a.data_ptr(), lda, int(a_mn), a[0].numel(), 0,
                           b.data_ptr(), ldb, int(b_mn), b[0].numel(), 0,
                           mode, alpha, c.data_ptr(), c_code, N, M * N, 0,
                           bias_t.data_ptr() if bias_t is not None else None,
                           resid.data_ptr() if resid is not None else None,
                           aux.data_ptr() if aux is not None else None)
    assert st == 0, lib.wp_last_error().decode()
    torch.cuda.synchronize()
    if mode == EPI_STORE:
        ref = acc
    elif mode == EPI_ACCUM:
        ref = c0 + acc
    elif mode == EPI_RESID:
        ref = resid.float() + acc
    elif mode == EPI_GELU:
        pre = acc.to(c_dtype).float()
        torch.testing.assert_close(aux.float(), pre, rtol=2e-2 if c_code else 1e-4, atol=2e-2 if c_code else 1e-4)
        ref = gelu(pre)
    else:
        ref = acc * gelu_grad(aux0)
    return c.float(), ref


LAYOUTS = [(False, False), (False, True), (True, False), (True, True)]


@pytest.mark.parametrize("a_mn,b_mn", LAYOUTS)
@pytest.mark.parametrize("shape", [(256, 512, 256), (128, 256, 64), (200, 304, 136), (384, 1000, 512)])
def test_tc_layouts(a_mn, b_mn, shape):
    M, N, K = shape
    out, ref = run(M, N, K, a_mn, b_mn, torch.bfloat16, c_dtype=torch.float32)
    # bf16 inputs, fp32 accumulate: the reference uses the same bf16-rounded inputs.
    torch.testing.assert_close(out, ref, rtol=1e-3, atol=1e-3 * K ** 0.5)


@pytest.mark.parametrize("mode", [EPI_STORE, EPI_ACCUM, EPI_RESID, EPI_GELU, EPI_DGELU])
def test_tc_epilogues(mode):
    c_dtype = torch.float32 if mode == EPI_ACCUM else torch.bfloat16
    out, ref = run(256, 768, 512, False, False, torch.bfloat16, mode=mode, bias=mode != EPI_DGELU,
                   c_dtype=c_dtype)
    tol = 1e-3 if c_dtype == torch.float32 else 2e-2
    torch.testing.assert_close(out, ref, rtol=tol, atol=tol * 8)


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True)])
@pytest.mark.parametrize("mode", [EPI_STORE, EPI_ACCUM, EPI_RESID, EPI_GELU, EPI_DGELU])
@pytest.mark.parametrize("shape", [(320, 1000, 136), (512, 776, 128), (1024, 384, 256)])
def test_tc_pair_tma_epilogue_ragged(a_mn, b_mn, mode, shape):
    """CTA-pair kernel with the TMA-store epilogue: every fused mode, the
    three operand layouts of the linear layers, ragged M / N edges (clipped
    stores, zero-filled residual / GELU-input loads)."""
    M, N, K = shape
    c_dtype = torch.float32 if mode == EPI_ACCUM else torch.bfloat16
    out, ref = run(M, N, K, a_mn, b_mn, torch.bfloat16, mode=mode, bias=mode != EPI_DGELU, c_dtype=c_dtype)
    tol = 1e-3 if c_dtype == torch.float32 else 2e-2
    torch.testing.assert_close(out, ref, rtol=tol, atol=tol * 8)


@pytest.mark.parametrize("shape", [(2048, 2048, 8192), (768, 512, 4096), (1024, 640, 2112), (6144, 2048, 16384),
                                   (1536, 512, 16384)])
def test_tc_pair_split_k_accumulation(shape):
    """Weight-gradient shapes whose tile count underfills the last wave of SM
    pairs run split-K: partial tiles reduce-add into the fp32 gradient."""
    M, N, K = shape
    out, ref = run(M, N, K, True, True, torch.bfloat16, mode=EPI_ACCUM, c_dtype=torch.float32)
    torch.testing.assert_close(out, ref, rtol=1e-3, atol=2e-3 * K ** 0.5)


@pytest.mark.parametrize("which", ["logits", "dgrad", "wgrad"])
def test_lm_head_vocab_50304(which):
    """The GPT-1.3B LM head at its own shapes (V = 50304 = 196.5 x 256: a
    ragged last N tile for the logits, a ragged last K block for the data
    gradient, a ragged last M tile for the fp32 weight gradient); T = 2048
    tokens, h = 2048."""
    T, h, V = 2048, 2048, 50304
    if which == "logits":   # logits[T, V] = LN[T, h] @ wte[V, h]^T, bf16 store
        out, ref = run(T, V, h, False, False, torch.bfloat16)
        torch.testing.assert_close(out, ref, rtol=2e-2, atol=2e-2 * 8)
    elif which == "dgrad":  # dLN[T, h] = dlogits[T, V] @ wte[V, h]
        out, ref = run(T, h, V, False, True, torch.bfloat16, c_dtype=torch.float32)
        torch.testing.assert_close(out, ref, rtol=1e-3, atol=2e-3 * V ** 0.5)
    else:                   # dwte[V, h] += dlogits^T @ LN  (both MN-major over T)
        out, ref = run(V, h, T, True, True, torch.bfloat16, mode=EPI_ACCUM, c_dtype=torch.float32)
        torch.testing.assert_close(out, ref, rtol=1e-3, atol=2e-3 * T ** 0.5)


lib.wp_debug_gemm_colsum.restype = C.c_int
lib.wp_debug_gemm_colsum.argtypes = [C.c_int] * 4 + [C.c_void_p, C.c_int64, C.c_int] * 2 + \
    [C.c_int, C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("M,N,K", [(512, 1024, 256), (320, 1000, 128), (8192, 8192, 2048)])
def test_gemm_fused_bias_grad_colsum(dtype, M, N, K):
    """dU = (dY W) * gelu'(U) with colsum += sum_rows(dU) fused into the
    epilogue (CTA-pair kernel; a separate pass elsewhere), vs torch fp32."""
    code = 1 if dtype == torch.bfloat16 else 0
    a = torch.randn(M, K, device="cuda").to(dtype)
    b = torch.randn(K, N, device="cuda").to(dtype)       # W stored [K, N]: N-major B
    aux = torch.randn(M, N, device="cuda").to(dtype)
    c = torch.empty(M, N, device="cuda", dtype=dtype)
    cs0 = torch.randn(N, device="cuda")
    cs = cs0.clone()
    st = lib.wp_debug_gemm_colsum(M, N, K, code, a.data_ptr(), K, 0, b.data_ptr(), N, 1, EPI_DGELU, c.data_ptr(),
                                  code, N, aux.data_ptr(), cs.data_ptr())
    assert st == 0, lib.wp_last_error().decode()
    ref = (a.float() @ b.float()) * gelu_grad(aux.float())
    tol = 2e-2 if code else 1e-4
    torch.testing.assert_close(c.float(), ref, rtol=tol, atol=tol * 8)
    # bf16 path sums the fp32 epilogue values; fp32 path sums the stored C
    got, want = cs - cs0, ref.sum(0)
    assert ((got - want).norm() / want.norm()).item() < (5e-3 if code else 1e-5)


def test_tc_pair_fp32_store_and_alpha():
    out, ref = run(384, 640, 192, False, True, torch.bfloat16, c_dtype=torch.float32, alpha=0.5, bias=True)
    torch.testing.assert_close(out, ref, rtol=1e-3, atol=1e-2)


def test_tc_batched_alpha():
    out, ref = run(128, 128, 64, False, False, torch.bfloat16, batch=6, alpha=0.125, c_dtype=torch.float32)
    torch.testing.assert_close(out, ref, rtol=1e-3, atol=1e-2)


@pytest.mark.parametrize("a_mn,b_mn", LAYOUTS)
@pytest.mark.parametrize("mode", [EPI_STORE, EPI_ACCUM, EPI_RESID, EPI_GELU, EPI_DGELU])
def test_simt_fp32(a_mn, b_mn, mode):
    out, ref = run(96, 130, 70, a_mn, b_mn, torch.float32, mode=mode, bias=mode != EPI_ACCUM, batch=2)
    torch.testing.assert_close(out, ref, rtol=1e-5, atol=1e-4)


def test_tc_large_throughput_sanity():
    """One big K-major GEMM: correctness at scale (the bench measures speed)."""
    M, N, K = 4096, 6144, 2048
    out, ref = run(M, N, K, False, False, torch.bfloat16, c_dtype=torch.float32)
    torch.testing.assert_close(out, ref, rtol=1e-3, atol=5e-2)


def _raw(M, N, K, a, lda, a_mn, b, ldb, b_mn, c, causal, nb=1, ab=0, bb=0, cb=0, in_code=1, c_code=0):
    fn = lib.wp_debug_gemm_causal
    st = fn(M, N, K, nb, 1, in_code, a.data_ptr(), lda, int(a_mn), ab, 0, b.data_ptr(), ldb, int(b_mn), bb, 0,
            0, 1.0, c.data_ptr(), c_code, N, cb, 0, None, None, None, causal)
    assert st == 0, lib.wp_last_error().decode()
    torch.cuda.synchronize()


lib.wp_debug_gemm_causal.restype = C.c_int
lib.wp_debug_gemm_causal.argtypes = lib.wp_debug_gemm.argtypes + [C.c_int]
CAUSAL_SKIP_UPPER, CAUSAL_K_UP_TO_ROW, CAUSAL_K_FROM_ROW = 1, 2, 3


def causal_p(s, nb, dtype):
    """Lower-triangular 'probabilities' with NaN beyond each row's 128-wide
    tile -- memory the causal GEMMs must never read."""
    p = torch.rand(nb, s, s, device="cuda").tril()
    q = torch.arange(s, device="cuda")[:, None]
    j = torch.arange(s, device="cuda")[None, :]
    p[:, (j >= (q // 128 + 1) * 128).expand(s, s)] = float("nan")
    return p.to(dtype)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_causal_modes(dtype):
    s, d, nb = 384, 128, 2
    in_code = 1 if dtype == torch.bfloat16 else 0
    q = torch.randn(nb, s, d, device="cuda").to(dtype)
    k = torch.randn(nb, s, d, device="cuda").to(dtype)
    # S = Q K^T with upper tiles skipped: lower triangle must match
    c = torch.zeros(nb, s, s, device="cuda")
    _raw(s, s, d, q, d, False, k, d, False, c, CAUSAL_SKIP_UPPER, nb, s * d, s * d, s * s, in_code)
    ref = q.float() @ k.float().transpose(1, 2)
    tri = torch.ones(s, s, device="cuda").tril().bool()
    tol = 2e-2 if in_code else 1e-4
    torch.testing.assert_close(c[:, tri], ref[:, tri], rtol=tol, atol=tol)
    # O = P V reading keys only up to each row tile's end
    p = causal_p(s, nb, dtype)
    v = torch.randn(nb, s, d, device="cuda").to(dtype)
    o = torch.zeros(nb, s, d, device="cuda")
    _raw(s, d, s, p, s, False, v, d, True, o, CAUSAL_K_UP_TO_ROW, nb, s * s, s * d, s * d, in_code)
    pz = torch.nan_to_num(p.float(), nan=0.0)
    torch.testing.assert_close(o, pz @ v.float(), rtol=tol, atol=tol * 4)
    # dV = P^T dO with queries starting at each key tile
    do = torch.randn(nb, s, d, device="cuda").to(dtype)
    dv = torch.zeros(nb, s, d, device="cuda")
    _raw(s, d, s, p, s, True, do, d, True, dv, CAUSAL_K_FROM_ROW, nb, s * s, s * d, s * d, in_code)
    torch.testing.assert_close(dv, pz.transpose(1, 2) @ do.float(), rtol=tol, atol=tol * 4)


def test_tc_narrow_n_tile():
    """N <= 128 selects the 128-wide tile; every layout."""
    for a_mn, b_mn in LAYOUTS:
        out, ref = run(384, 128, 320, a_mn, b_mn, torch.bfloat16, c_dtype=torch.float32)
        torch.testing.assert_close(out, ref, rtol=1e-3, atol=2e-2)
        out, ref = run(256, 72, 128, a_mn, b_mn, torch.bfloat16, c_dtype=torch.float32)
        torch.testing.assert_close(out, ref, rtol=1e-3, atol=2e-2)
