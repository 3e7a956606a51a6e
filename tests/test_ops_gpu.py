"""HBM-bound stage kernels vs a torch fp32 reference of the same op (GPU):
LayerNorm forward and the fused backward (dx with residual, dw / db partial
sums), and the vectorised fused cross-entropy (loss + dlogits in place), at
the tiny and the GPT-1.3B shapes."""
import ctypes as C

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2308_15762_b200 import _native  # noqa: E402

lib = _native.lib
P = C.c_void_p
lib.wp_debug_layernorm.restype = C.c_int
lib.wp_debug_layernorm.argtypes = [C.c_int, C.c_int, C.c_int] + [P] * 11
lib.wp_debug_xent.restype = C.c_int
lib.wp_debug_xent.argtypes = [C.c_int, P, P, P, C.c_int, C.c_int, C.c_float, C.c_float]


def ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("T,h,resid", [(256, 256, True), (1000, 1024, False), (8192, 2048, True), (64, 4096, True)])
def test_layernorm_fwd_bwd(dtype, T, h, resid):
    code = 1 if dtype == torch.bfloat16 else 0
    g = torch.Generator(device="cuda").manual_seed(3)
    x = (torch.randn(T, h, device="cuda", generator=g) * 2 + 0.5).to(dtype)
    w = torch.randn(h, device="cuda", generator=g)
    b = torch.randn(h, device="cuda", generator=g)
    dy = torch.randn(T, h, device="cuda", generator=g).to(dtype)
    dres = torch.randn(T, h, device="cuda", generator=g).to(dtype) if resid else None
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    mean = torch.empty(T, device="cuda")
    rstd = torch.empty(T, device="cuda")
    dw0 = torch.randn(h, device="cuda", generator=g)  # gradients accumulate (+=)
    db0 = torch.randn(h, device="cuda", generator=g)
    dw, db = dw0.clone(), db0.clone()
    st = lib.wp_debug_layernorm(code, T, h, ptr(x), ptr(w), ptr(b), ptr(y), ptr(mean), ptr(rstd), ptr(dy),
                                ptr(dres), ptr(dx), ptr(dw), ptr(db))
    assert st == 0, lib.wp_last_error().decode()
    xf = x.float().requires_grad_(True)
    wf = w.clone().requires_grad_(True)
    bf = b.clone().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xf, (h,), wf, bf, eps=1e-5)
    yr.backward(dy.float())
    tol = 1e-4 if code == 0 else 2e-2
    torch.testing.assert_close(y.float(), yr.detach(), rtol=tol, atol=tol)
    want_dx = xf.grad + (dres.float() if resid else 0)
    torch.testing.assert_close(dx.float(), want_dx, rtol=tol, atol=tol * 4)
    # dw / db: fp32 sums over T rows of act-dtype inputs -> normwise bound
    for got, base, ref in ((dw, dw0, wf.grad), (db, db0, bf.grad)):
        err = (got - base - ref).norm() / ref.norm()
        assert err < (1e-5 if code == 0 else 1e-3), err


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("T,V", [(256, 1024), (1030, 50304), (64, 1000)])
def test_xent(dtype, T, V):
    code = 1 if dtype == torch.bfloat16 else 0
    g = torch.Generator(device="cuda").manual_seed(5)
    logits = (torch.randn(T, V, device="cuda", generator=g) * 3).to(dtype)
    labels = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
    l0 = logits.float().clone().requires_grad_(True)
    loss = torch.full((1,), 0.25, device="cuda")
    scale = 1.0 / T
    st = lib.wp_debug_xent(code, ptr(logits), ptr(labels), ptr(loss), T, V, scale, scale)
    assert st == 0, lib.wp_last_error().decode()
    ref = torch.nn.functional.cross_entropy(l0, labels.long(), reduction="mean")
    ref.backward()
    ref = ref.detach()
    assert abs(float(loss) - 0.25 - float(ref)) <= 1e-5 * max(1.0, abs(float(ref))) * (1 if code == 0 else 10)
    tol = 1e-6 if code == 0 else 4e-3 / T
    torch.testing.assert_close(logits.float(), l0.grad, rtol=2e-2 if code else 1e-4, atol=tol)
