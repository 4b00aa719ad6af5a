"""The energy kernels' call-free IEEE division / reciprocal / square root (pairmath.cuh
div_rn_fast, rcp_rn_fast, sqrt_rn_fast) are bit-identical to __fdiv_rn / __fsqrt_rn over the
kernels' operand domain -- the premise of bit-identical per-pair energies with the oracle
(DESIGN.md section 5)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2405_01420_b200", "csrc")


def _build(tmp):
    exe = os.path.join(tmp, "ieee_fast_check")
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-fmad=false",
           f"-I{CSRC}", f"-I{os.path.join(ROOT, 'include')}", os.path.join(ROOT, "tests", "cuda", "ieee_fast_check.cu"),
           "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_ieee_fast_check_compiles(tmp_path):
    """nvcc cross-compiles the checker here (no GPU needed)."""
    assert os.path.exists(_build(str(tmp_path)))


@pytest.mark.gpu
def test_ieee_fast_paths_bit_exact(gpu, tmp_path):
    exe = _build(str(tmp_path))
    r = subprocess.run([exe, str(1 << 28)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("mismatches 0 "), r.stdout
