"""Host-side section timing of DomainDecomposition.repartition (torchrun, N GPUs).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/dd_repart_timing.py [config]
"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_01420_b200 import dd as DD  # noqa: E402
from paper_2405_01420_b200 import systems  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "water12m"
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    s = systems.make(cfg)
    d = DD.DomainDecomposition(s, rank, world, lambda sy, pbc: DD.NbxEngine(sy, local, pbc), device=dev,
                               halo=os.environ.get("NBX_DD_HALO", "p2p"))
    xg = torch.from_numpy(s.x).to(dev)
    d.repartition(xg)
    d.step(None, step=1)
    runs = []
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    for it in range(6):
        # moved coordinates every other repartition (as between two searches of an MD run)
        xr = xg if it % 2 == 0 else xg + 0.02 * torch.randn(xg.shape, device=dev, generator=g)
        d.timing = {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if os.environ.get("NBX_REPART", "global") == "device" and d.halo == "p2p":
            d.repartition(x_home=d.x_ext[:d.n_home])  # device-side neighbour-only repartition
        else:
            d.repartition(xr)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        d.step(None, step=1, prune=False)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        runs.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), dict(d.timing)))
    for r in range(world):
        dist.barrier()
        if rank == r:
            for tr, ts, tim in runs:
                print(f"rank {rank}: repartition {tr:.2f} ms, first step after {ts:.2f} ms: "
                      + ", ".join(f"{k} {1e3 * v:.2f}" for k, v in tim.items()), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
