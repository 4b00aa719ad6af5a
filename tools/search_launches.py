"""Two grid+search calls on a config (the second one is steady state: single pass with the
capacities of the first).  Run under `ncu --metrics gpu__time_duration.sum` for the launch list.

    python tools/search_launches.py [config]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_01420_b200 import nbx, systems  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "water12m"
s = systems.make(cfg)
nb = nbx.Nonbonded(s)
x = torch.from_numpy(s.x).cuda()
for k in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nb.search(x)
    torch.cuda.synchronize()
    print(f"search {k}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
