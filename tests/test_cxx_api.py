"""The C++ drop-in (include/wavepipe/*.hpp, reference include names) compiles
and links against libwavepipe.so on CPU; on a GPU the demo runs
wavepipe::train_step and feeds the measured trace to bubble_ratio and
trace_to_gantt unchanged."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2308_15762_b200")
EXE = os.path.join(ROOT, "build", "train_step_demo")


def _build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cxx", "train_step_demo.cpp"), "-L" + LIBDIR, "-lwavepipe",
                    "-Wl,-rpath," + LIBDIR, "-o", EXE], check=True, capture_output=True, text=True)


def test_cxx_api_compiles_and_links():
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_cxx_train_step_on_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    _build()
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("step ") == 3
