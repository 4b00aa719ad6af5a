"""Search steps under NVML polling: device time of consecutive search steps (grid + search +
prune + force + F op) with an nvidia-smi sampler polling every 50 ms, and the library's device
allocations per step (cudaMalloc/cudaFree contend with NVML for the driver lock).

    python tools/search_stall.py [config] [n_searches]
"""
import json
import os
import subprocess
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_01420_b200 import nbx, systems  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "water12m"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
s = systems.make(cfg)
nb = nbx.Nonbonded(s)
x = torch.from_numpy(s.x).cuda()
f = torch.empty_like(x)
v = torch.randn(x.shape, device="cuda") * 3e-4
for poll in (False, True):
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "50"],
                           stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL) if poll else None
    ms, allocs = [], []
    for k in range(n):
        x += v
        a0 = nb.alloc_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nb.step(x, f, 0)  # a search step
        for j in range(1, 4):
            nb.step(x, f, j)  # and a few plain steps queued behind it, as in an MD run
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        allocs.append(nb.alloc_count() - a0)
    if smi:
        smi.terminate()
        smi.wait()
    a = np.array(ms)
    print(json.dumps({"config": cfg, "nvidia_smi_50ms": poll, "n": n, "median_ms": float(np.median(a)),
                      "max_ms": float(a.max()), "p90_ms": float(np.percentile(a, 90)),
                      "over_2x_median": int((a > 2 * np.median(a)).sum()), "allocs": allocs}), flush=True)
