"""Peer-halo guard rails on one GPU (a world of one rank: the region is its own, no IPC).

nbx_peer_set_halo validates every halo entry on the device: an owner rank or owner home index
outside the peer regions is never dereferenced by the step kernels and is reported through
nbx_peer_status (2); dd.py's check_peer raises on it."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(cap=64):
    import torch

    from paper_2405_01420_b200 import dd as DD
    from paper_2405_01420_b200 import systems
    s = systems.water_box(1000, seed=3, coulomb="ewald", rc=0.9, rlist_outer=1.0, rlist_inner=0.92)
    eng = DD.NbxEngine(s, 0, [1, 1, 1])
    h = eng.peer_init(0, 1, cap)
    eng.peer_open(h)
    x = torch.from_numpy(s.x).cuda()
    gid = torch.arange(s.natoms, dtype=torch.int32, device="cuda")
    box = np.asarray(s.box, np.float32)
    eng.grid_build(0, x[:40], gid[:40], np.zeros(3, np.float32), box)
    eng.search(0)
    eng.grid_build(1, x[40:42], gid[40:42], np.zeros(3, np.float32), box)
    eng.search(1)
    return eng


def test_peer_invalid_halo_map_is_reported(gpu):
    import torch
    eng = _setup()
    owner = torch.tensor([0, 3], dtype=torch.int32, device="cuda")  # rank 3 does not exist
    home = torch.tensor([0, 1], dtype=torch.int32, device="cuda")
    shift = torch.zeros((2, 3), dtype=torch.float32, device="cuda")
    eng.peer_set_halo(owner, home, shift)
    torch.cuda.synchronize()
    assert eng.peer_status() == 2


def test_peer_home_index_beyond_capacity_is_reported(gpu):
    import torch
    eng = _setup(cap=64)
    owner = torch.tensor([0, 0], dtype=torch.int32, device="cuda")
    home = torch.tensor([0, 64], dtype=torch.int32, device="cuda")  # == capacity
    shift = torch.zeros((2, 3), dtype=torch.float32, device="cuda")
    eng.peer_set_halo(owner, home, shift)
    torch.cuda.synchronize()
    assert eng.peer_status() == 2
    # a valid map clears the report
    eng.peer_set_halo(owner, torch.tensor([0, 1], dtype=torch.int32, device="cuda"), shift)
    torch.cuda.synchronize()
    assert eng.peer_status() == 0
