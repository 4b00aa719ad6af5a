"""Search-step timing with moving coordinates: device time (CUDA events) and host time of
consecutive nbx_search calls, each after a small displacement (diagnostics for bench.py)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2405_01420_b200 import nbx, systems  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "water12m"
s = systems.make(cfg)
nb = nbx.Nonbonded(s, device=0)
x = torch.from_numpy(s.x).cuda()
rng = np.random.default_rng(1)
out = []
for it in range(8):
    if it:
        x += torch.from_numpy(rng.normal(scale=0.01, size=s.x.shape).astype(np.float32)).cuda()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    nb.search(x)
    e1.record()
    th = time.perf_counter() - t0
    torch.cuda.synchronize()
    out.append({"it": it, "device_ms": e0.elapsed_time(e1), "host_ms": 1e3 * th, **nb.list_sizes()})
    print(json.dumps(out[-1]), flush=True)
