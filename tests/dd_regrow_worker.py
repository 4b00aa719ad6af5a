"""torchrun worker for tests/test_dd_gpu.py::test_dd_peer_capacity_regrow_one_gpu.

    torchrun --nproc-per-node 2 tests/dd_regrow_worker.py <out.npz>      (ranks share cuda:0, gloo)

After a global partition and a device-side repartition, the water molecules are moved rigidly
towards x = 0 (oxygen x -> 0.75 x): domain 0 of the 2x1x1 split then holds ~2/3 of the atoms,
more than the peer regions' capacity (NBX_PEER_CAP_FACTOR=1.0: ~1.25x the first partition's
largest home set).  The next
device-side repartition must report the overflow, fall back to the global partition from an
all-gather of the home sets, re-create the peer regions larger on all ranks together (ADVICE
r1), and still give the single-GPU forces and energies.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2405_01420_b200 import dd as DD  # noqa: E402
from paper_2405_01420_b200 import nbx, systems  # noqa: E402
from tests.dd_gpu_worker import gather_home  # noqa: E402


def main():
    out = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo")
    s = systems.make("water12m", 90000)
    d = DD.DomainDecomposition(s, rank, world, lambda sy, pbc: DD.NbxEngine(sy, 0, pbc), device=dev, halo="p2p")
    xg = torch.from_numpy(s.x).to(dev)
    d.repartition(xg)
    d.step(None, step=1)
    d.repartition(x_home=d.x_ext[:d.n_home])  # device path, no overflow
    cap0 = d._peer_cap
    # squeeze the molecules (rigidly, by their oxygen) towards x = 0: domain 0 gains atoms
    # beyond the capacity; molecules stay intact, so no atom pair comes unphysically close
    xs = s.x.astype(np.float64).copy()
    ox = xs[0::3, 0]
    for k in range(3):
        xs[k::3, 0] += (0.75 - 1.0) * ox
    xsq = torch.from_numpy(xs.astype(np.float32)).to(dev)
    d.repartition(x_home=xsq[d.home_gid.long()])
    f, (e, vir) = d.step(None, step=100, energy=True, virial=True, prune=False)
    torch.cuda.synchronize()
    d.check_peer()
    G, F = gather_home(d, f.clone(), world, dev, s.natoms)
    nmax = torch.tensor([d.n_home], dtype=torch.int64, device=dev)
    nmax = int(d._all_reduce(nmax, op=dist.ReduceOp.MAX)[0])
    if rank == 0:
        X = xsq
        nb = nbx.Nonbonded(s, device=0)
        nb.search(X)
        f1, (e1, v1) = nb.forces(X, energy=True, virial=True)
        np.savez(out, f=F, gids=G, e=e, vir=vir, f_ref=f1.cpu().numpy(), e_ref=e1, vir_ref=v1, cap0=cap0,
                 cap1=d._peer_cap, nmax=nmax, fallback=d.repartitions["fallback"], peer_inits=d.peer_inits,
                 natoms=s.natoms)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
