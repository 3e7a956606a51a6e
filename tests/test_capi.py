"""The C-ABI library loads and exports every symbol include/*.h declares (CPU;
no compute calls).  Error codes follow the reference CLI taxonomy."""
import ctypes as C
import os
import re

import paper_2308_15762_b200 as wp
from paper_2308_15762_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    inc = os.path.join(ROOT, "include")
    for fn in os.listdir(inc):
        if fn.endswith(".h"):
            text = open(os.path.join(inc, fn)).read()
            text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
            names |= set(re.findall(r"\b(wp_[a-z0-9_]+)\s*\(", text))
    return names


def test_every_declared_symbol_is_exported():
    decl = declared_symbols()
    assert len(decl) >= 40
    lib = C.CDLL(_native.LIB_PATH)
    missing = [n for n in sorted(decl) if not hasattr(lib, n)]
    assert not missing, missing
    assert not _native.MISSING
    assert set(_native.EXPORTED) == decl


def test_error_codes_and_messages():
    out = _native.wp_config()
    assert _native.lib.wp_make_config(4, 4, 2, 2, 1, C.byref(out)) == _native.WP_ERR_CONFIG
    assert b"B must be >= P" in _native.lib.wp_last_error()
    assert _native.lib.wp_make_config(4, 4, 8, 2, 1, C.byref(out)) == _native.WP_OK
    assert (out.devices, out.microbatches, out.waves, out.stages) == (4, 8, 2, 16)
    assert _native.lib.wp_parse(b"{not json", C.byref(C.c_void_p())) == _native.WP_ERR_CONFIG


def test_runtime_refuses_without_gpu_or_invalid_list():
    """No CPU fallback: without a CUDA device the runtime reports WP_ERR_CUDA."""
    import torch
    if torch.cuda.is_available():
        return
    lst = wp.generate_schedule(wp.make_config(wp.Scheme.Hanayo, 2, 4, 2))
    try:
        wp.Runtime(wp.ModelDesc(), lst)
    except wp.schedule.ScheduleError as e:  # pragma: no cover - wrong class
        raise AssertionError(e)
    except _native.CudaError as e:
        assert e.code == _native.WP_ERR_CUDA
    else:  # pragma: no cover
        raise AssertionError("runtime created without a GPU")
