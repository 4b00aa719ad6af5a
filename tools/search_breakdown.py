"""Search-step breakdown on a small box: host wall time of nbx_grid_build and nbx_search
(each ends in a host synchronisation), and device time of each via CUDA events.  Under
`ncu --metrics gpu__time_duration.sum` the same script gives the per-kernel launch list.

    python tools/search_breakdown.py [config] [reps] [natoms]
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2405_01420_b200 import nbx, systems  # noqa: E402
from paper_2405_01420_b200.nbx import LIST_LOCAL, _dev_ptr, _ptr, _stream, check, lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "rnase24k"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
s = systems.make(cfg, int(sys.argv[3]) if len(sys.argv) > 3 else None)
nb = nbx.Nonbonded(s, device=0)
x = torch.from_numpy(s.x).cuda()
nb.search(x)
nb.search(x)
torch.cuda.synchronize()
st = _stream(torch, None)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
hg, hs, dg, ds = [], [], [], []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record()
    check(lib().nbx_grid_build(nb.ctx.h, 0, nb.n, _dev_ptr(x), None, _ptr(nb._lo), _ptr(nb.box), st))
    ev[1].record()
    t1 = time.perf_counter()
    check(lib().nbx_search(nb.ctx.h, LIST_LOCAL, st))
    ev[2].record()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    hg.append(t1 - t0)
    hs.append(t2 - t1)
    dg.append(ev[0].elapsed_time(ev[1]))
    ds.append(ev[1].elapsed_time(ev[2]))
med = lambda a: float(np.median(a))  # noqa: E731
print(json.dumps({"config": cfg, "natoms": s.natoms, "host_grid_ms": 1e3 * med(hg), "host_search_ms": 1e3 * med(hs),
                  "dev_grid_ms": med(dg), "dev_search_ms": med(ds), **nb.list_sizes()}))
