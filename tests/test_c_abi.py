"""The C-ABI from plain C (tests/c_abi/nbx_c_smoke.c): compiles with gcc against
include/nbx.h and links libnbx.so (CPU); runs the reference cadence with PME and the update
on a B200 and checks Newton's third law, energy-step/force-step agreement and error
reporting (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c_abi", "nbx_c_smoke.c")
LIBDIR = os.path.join(ROOT, "paper_2405_01420_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build(tmp_path):
    exe = str(tmp_path / "nbx_c_smoke")
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Werror", "-o", exe, SRC, f"-I{ROOT}/include", f"-I{CUDA}/include",
           f"-L{LIBDIR}", "-lnbx", f"-Wl,-rpath,{LIBDIR}", f"-L{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{CUDA}/lib64",
           "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_consumer_compiles_and_links(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libnbx.so")):
        pytest.skip("libnbx.so not built")
    exe = build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_c_consumer_runs(gpu, tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "nbx_c_smoke ok" in r.stdout
