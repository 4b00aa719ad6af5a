"""Domain decomposition on real GPUs (NCCL), N = 2 / 4 / 8 as many as are visible.

DD forces, energies and virial == the single-GPU engine on the same coordinates, after a
search step and after a moved-atoms prune step.  Skipped on a 1-GPU box (the host logic is
covered on CPU by tests/test_dd.py)."""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

from tests.helpers import assert_energies, assert_forces, assert_virial

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("halo", ["nccl", "p2p"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_dd_matches_single_gpu(gpu, world, halo):
    """halo=p2p: force-only steps through the NVLink peer-memory halo (csrc/peer.cu)."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    natoms = 150000 if world < 8 else 300000
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "dd.npz")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(29500 + world),
               os.path.join(ROOT, "tests", "dd_gpu_worker.py"), "water12m", str(natoms), out, halo]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
        d = np.load(out)
    assert np.array_equal(np.sort(d["gids"]), np.arange(int(d["natoms"])))
    assert_forces(d["f"], d["f_ref"])
    assert_energies(d["e"], d["e_ref"])
    assert_virial(d["vir"], d["vir_ref"])
    assert_forces(d["f2"], d["f2_ref"])
    assert_energies(d["e2"], d["e2_ref"])
    assert_virial(d["vir2"], d["vir2_ref"])
    assert_forces(d["fa"], d["f_ref"])
    assert_forces(d["fb"], d["f2_ref"])
    assert_forces(d["fb2"], d["f2_ref"])


@pytest.mark.parametrize("config", ["stmv_tab", "grappa1.5m", "rnase24k_lb"])
@pytest.mark.parametrize("world", [2, 4])
def test_dd_paper_flavours(gpu, world, config):
    """The paper's kernel flavours through the DD path (NVLink peer halo): tabulated Ewald +
    force-switch LJ (STMV flavour), tabulated Ewald + LB combination rule (Grappa flavour), and
    LB on the protein-like box; forces, energies and virial == the single-GPU engine."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    natoms = 60000 if config == "rnase24k_lb" else 150000
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "dd.npz")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(29520 + world),
               os.path.join(ROOT, "tests", "dd_gpu_worker.py"), config, str(natoms), out, "p2p"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
        d = np.load(out)
    assert np.array_equal(np.sort(d["gids"]), np.arange(int(d["natoms"])))
    assert_forces(d["f"], d["f_ref"])
    assert_energies(d["e"], d["e_ref"])
    assert_virial(d["vir"], d["vir_ref"])
    assert_forces(d["fa"], d["f_ref"])
    assert_forces(d["fb"], d["f2_ref"])
