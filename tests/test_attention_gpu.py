"""Fused (flash) attention kernels vs a torch fp32 reference (GPU)."""
import ctypes as C
import math

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2308_15762_b200 import _native  # noqa: E402

lib = _native.lib
lib.wp_debug_flash_fwd.restype = C.c_int
lib.wp_debug_flash_fwd.argtypes = [C.c_int] * 5 + [C.c_void_p] * 3


def reference(qkv, mbs, seq, heads, d, causal):
    h = heads * d
    x = qkv.float().view(mbs, seq, 3, heads, d)
    q, k, v = (x[:, :, i].transpose(1, 2) for i in range(3))  # [mbs, heads, seq, d]
    s = q @ k.transpose(-1, -2) / math.sqrt(d)
    if causal:
        s = s.masked_fill(torch.ones(seq, seq, device=s.device, dtype=torch.bool).triu(1), float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ v
    return o.transpose(1, 2).reshape(mbs * seq, h), lse / math.log(2.0)


@pytest.mark.parametrize("mbs,seq,heads,d,causal", [(2, 128, 4, 64, 1), (2, 256, 2, 128, 1), (1, 512, 3, 128, 0),
                                                     (2, 384, 2, 64, 0), (1, 1024, 2, 128, 1)])
def test_flash_fwd(mbs, seq, heads, d, causal):
    torch.manual_seed(0)
    h = heads * d
    qkv = (torch.randn(mbs * seq, 3 * h, device="cuda") * 1.5).bfloat16()
    ctx = torch.empty(mbs * seq, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(mbs, heads, seq, device="cuda")
    assert lib.wp_debug_flash_fwd(mbs, seq, heads, d, causal, qkv.data_ptr(), ctx.data_ptr(), lse.data_ptr()) == 0, \
        lib.wp_last_error()
    ref_o, ref_lse = reference(qkv, mbs, seq, heads, d, causal)
    torch.testing.assert_close(ctx.float(), ref_o, rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(lse, ref_lse, rtol=1e-3, atol=1e-3)


lib.wp_debug_flash_bwd.restype = C.c_int
lib.wp_debug_flash_bwd.argtypes = [C.c_int] * 5 + [C.c_void_p] * 7


@pytest.mark.parametrize("mbs,seq,heads,d,causal", [(2, 128, 4, 64, 1), (2, 256, 2, 128, 1), (1, 512, 3, 128, 0),
                                                     (2, 384, 2, 64, 0), (1, 1024, 2, 128, 1)])
def test_flash_bwd(mbs, seq, heads, d, causal):
    torch.manual_seed(1)
    h = heads * d
    qkv = torch.randn(mbs * seq, 3 * h, device="cuda").bfloat16()
    ctx = torch.empty(mbs * seq, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(mbs, heads, seq, device="cuda")
    assert lib.wp_debug_flash_fwd(mbs, seq, heads, d, causal, qkv.data_ptr(), ctx.data_ptr(), lse.data_ptr()) == 0
    dout = torch.randn(mbs * seq, h, device="cuda").bfloat16()
    delta = torch.empty(mbs, heads, seq, device="cuda")
    dq_acc = torch.empty(mbs * seq, h, device="cuda")
    dqkv = torch.zeros(mbs * seq, 3 * h, device="cuda", dtype=torch.bfloat16)
    assert lib.wp_debug_flash_bwd(mbs, seq, heads, d, causal, qkv.data_ptr(), ctx.data_ptr(), dout.data_ptr(),
                                  lse.data_ptr(), delta.data_ptr(), dq_acc.data_ptr(), dqkv.data_ptr()) == 0, \
        lib.wp_last_error()
    x = qkv.float().requires_grad_(True)
    o, _ = reference(x, mbs, seq, heads, d, causal)
    o.backward(dout.float())
    ref = x.grad
    for part in range(3):
        got = dqkv[:, part * h:(part + 1) * h].float()
        want = ref[:, part * h:(part + 1) * h]
        err = (got - want).norm() / want.norm()
        assert err < 2e-2, (part, err.item())


lib.wp_debug_flash_bwd_bias.restype = C.c_int
lib.wp_debug_flash_bwd_bias.argtypes = [C.c_int] * 5 + [C.c_void_p] * 8


@pytest.mark.parametrize("mbs,seq,heads,d,causal", [(2, 256, 2, 128, 1), (2, 384, 2, 64, 0)])
def test_flash_bwd_fused_bias_grad(mbs, seq, heads, d, causal):
    """The QKV bias gradient the backward accumulates (column sums of dQKV,
    from the fp32 dK / dV accumulators and dQ) matches torch's dQKV.sum(0);
    it adds to what the buffer held."""
    torch.manual_seed(2)
    h = heads * d
    qkv = torch.randn(mbs * seq, 3 * h, device="cuda").bfloat16()
    ctx = torch.empty(mbs * seq, h, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(mbs, heads, seq, device="cuda")
    assert lib.wp_debug_flash_fwd(mbs, seq, heads, d, causal, qkv.data_ptr(), ctx.data_ptr(), lse.data_ptr()) == 0
    dout = torch.randn(mbs * seq, h, device="cuda").bfloat16()
    delta = torch.empty(mbs, heads, seq, device="cuda")
    dq_acc = torch.empty(mbs * seq, h, device="cuda")
    dqkv = torch.zeros(mbs * seq, 3 * h, device="cuda", dtype=torch.bfloat16)
    dbias = torch.full((3 * h,), 0.5, device="cuda")
    assert lib.wp_debug_flash_bwd_bias(mbs, seq, heads, d, causal, qkv.data_ptr(), ctx.data_ptr(), dout.data_ptr(),
                                       lse.data_ptr(), delta.data_ptr(), dq_acc.data_ptr(), dqkv.data_ptr(),
                                       dbias.data_ptr()) == 0, lib.wp_last_error()
    x = qkv.float().requires_grad_(True)
    o, _ = reference(x, mbs, seq, heads, d, causal)
    o.backward(dout.float())
    want = x.grad.sum(0) + 0.5
    err = (dbias - want).norm() / (want - 0.5).norm()
    assert err < 2e-2, err.item()

