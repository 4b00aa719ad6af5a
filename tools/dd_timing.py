"""Time DD repartition (search step) and regular steps per rank (torchrun)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2405_01420_b200 import dd as DD  # noqa: E402
from paper_2405_01420_b200 import systems  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
dev = torch.device("cuda", local)
s = systems.make(sys.argv[1] if len(sys.argv) > 1 else "water12m")
d = DD.DomainDecomposition(s, rank, world, lambda sy, pbc: DD.NbxEngine(sy, local, pbc), device=dev)
xg = torch.from_numpy(s.x).to(dev)
out = []
for it in range(4):
    dist.barrier()
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.repartition(xg)
    torch.cuda.synchronize()
    t_rep = time.perf_counter() - t
    x_home = d.x_ext[:d.n_home].clone()
    dist.barrier()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for k in range(1, 11):
        d.step(x_home, step=k)
    torch.cuda.synchronize()
    t_steps = (time.perf_counter() - t) / 10
    out.append((round(t_rep * 1e3, 2), round(t_steps * 1e3, 3)))
print(f"rank {rank}: n_home {d.n_home} n_ext {d.n_ext} (repartition ms, step ms):", out, flush=True)
dist.destroy_process_group()
