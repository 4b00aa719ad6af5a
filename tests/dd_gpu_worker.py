"""torchrun worker for tests/test_dd_gpu.py: DD over NCCL on N GPUs vs the single-GPU engine.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/dd_gpu_worker.py <config> <natoms> <out.npz> [nccl|p2p]

p2p: force-only steps go through the NVLink peer-memory halo (csrc/peer.cu) and are checked
as well; energy/virial steps always take the NCCL path.
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


def main():
    cfg, natoms, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    halo = sys.argv[4] if len(sys.argv) > 4 else "nccl"
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    s = systems.make(cfg, natoms)
    d = DD.DomainDecomposition(s, rank, world, lambda sy, pbc: DD.NbxEngine(sy, local, pbc), device=dev,
                                halo=halo)
    xg = torch.from_numpy(s.x).to(dev)
    d.repartition(xg)
    fa = d.step(None, step=1, prune=False).clone()  # force-only: the p2p path when halo=p2p
    f, (e, vir) = d.step(None, step=1, energy=True, virial=True, prune=False)
    f = f.clone()  # step() returns a view of the rank's force buffer
    # a second, non-search step with moved atoms (halo coordinates refreshed, prune on)
    rng = np.random.default_rng(3)
    disp = torch.from_numpy(rng.uniform(-0.01, 0.01, size=s.x.shape).astype(np.float32)).to(dev)
    x_home = d.x_ext[:d.n_home] + disp[d.home_gid.long()]
    fb = d.step(x_home, step=10, prune=True).clone()
    fb2 = d.step(x_home, step=11, prune=False).clone()  # a second step: inbox/flags reuse
    f2, (e2, vir2) = d.step(x_home, step=10, energy=True, virial=True, prune=True)
    torch.cuda.synchronize()
    d.check_peer()
    gids = [torch.zeros(0)] * world
    n = torch.tensor([d.n_home], device=dev)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    mx = int(max(int(v) for v in ns))
    pad = lambda t, w: torch.cat([t, torch.zeros((mx - t.shape[0],) + t.shape[1:], dtype=t.dtype, device=dev)])
    gl = [torch.zeros(mx, dtype=torch.int32, device=dev) for _ in range(world)]
    fl = [torch.zeros((mx, 3), dtype=torch.float32, device=dev) for _ in range(world)]
    fl2 = [torch.zeros((mx, 3), dtype=torch.float32, device=dev) for _ in range(world)]
    dist.all_gather(gl, pad(d.home_gid, 1))
    dist.all_gather(fl, pad(f.contiguous(), 1))
    dist.all_gather(fl2, pad(f2.contiguous(), 1))
    extra = {}
    for name, t in (("fa", fa), ("fb", fb), ("fb2", fb2)):
        lst = [torch.zeros((mx, 3), dtype=torch.float32, device=dev) for _ in range(world)]
        dist.all_gather(lst, pad(t.contiguous(), 1))
        extra[name] = lst
    if rank == 0:
        G = np.concatenate([gl[r][:int(ns[r])].cpu().numpy() for r in range(world)])
        F = np.zeros((s.natoms, 3))
        F2 = np.zeros((s.natoms, 3))
        F[G] = np.concatenate([fl[r][:int(ns[r])].cpu().numpy() for r in range(world)])
        F2[G] = np.concatenate([fl2[r][:int(ns[r])].cpu().numpy() for r in range(world)])
        FX = {}
        for name, lst in extra.items():
            FX[name] = np.zeros((s.natoms, 3))
            FX[name][G] = np.concatenate([lst[r][:int(ns[r])].cpu().numpy() for r in range(world)])
        # single-GPU reference with the same coordinates
        nb = nbx.Nonbonded(s, device=local)
        nb.search(xg)
        f1, (e1, v1) = nb.forces(xg, energy=True, virial=True)
        x2 = xg + disp
        nb.put_x(x2)
        nb.prune()
        f12, (e12, v12) = nb.forces(x2, energy=True, virial=True)
        np.savez(out, gids=G, f=F, e=e, vir=vir, f_ref=f1.cpu().numpy(), e_ref=e1, vir_ref=v1, f2=F2, e2=e2,
                 vir2=vir2, f2_ref=f12.cpu().numpy(), e2_ref=e12, vir2_ref=v12, natoms=s.natoms, **FX)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
