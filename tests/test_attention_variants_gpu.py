"""The attention kernels' A/B switches stay correct (GPU): the forward with
every polynomial-exp2 share (WP_FA_POLY) and the backward with dQ in two N=64
halves (WP_BW_DQ_HALVES=1) pass the same torch fp32 checks as the defaults.
The switches are read once per process, so each runs in a subprocess."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"WP_FA_POLY": "0"}, {"WP_FA_POLY": "2"}, {"WP_FA_POLY": "5"},
                                 {"WP_BW_DQ_HALVES": "1"}])
def test_attention_switch(env):
    out = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_attention_gpu.py"), "-q",
                          "-x", "-p", "no:cacheprovider"], capture_output=True, text=True, timeout=900, cwd=ROOT,
                         env=dict(os.environ, **env))
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
