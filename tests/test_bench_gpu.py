"""bench.py's GPU arm end to end (GPU): the default single-rank line, and the
multi-rank path `bench.py --gpus 2` spawning its own two ranks (here both on
cuda:0 through WP_BENCH_SHARE_GPU=1, the IPC transport between them) with
rank 0 printing one line that carries the measured and simulated bubble and
the P2P figures."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(args, env_extra=None):
    env = dict(os.environ, **(env_extra or {}))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


def test_single_rank_line():
    d = run_bench(["--model", "tiny-gpt", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"])
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    # (a tiny model's timed region may end before nvidia-smi's first sample)
    assert d["roofline"]["bound"] == "tensor" and "clocks" in d


def test_two_ranks_spawned_on_one_gpu():
    d = run_bench(["--gpus", "2", "--model", "tiny-gpt", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"],
                  {"WP_BENCH_SHARE_GPU": "1"})
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert "P=2" in d["config"]["schedule"]
    assert d["p2p"]["transport"] == "ipc" and d["p2p"]["messages"] > 0
    b = d["bubble"]
    assert 0.0 <= b["measured"] < 1.0 and 0.0 <= b["simulated_at_measured_costs"] < 1.0
    assert d["memory"]["landing_gb_max"] >= 0.0
