"""Row f2 measurement: force-kernel time and whole NB step (graph-replayed, as bench.py's
small-box path) with the list order (NBX_ENTRY_ORDER=0) and longest-first (=1), on the small
boxes the paper says the sort matters for and the large ones.

    python tools/time_entry_order.py <order> [config ...]     (one order per process: env read at create)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01420_b200 import nbx, systems  # noqa: E402


def timed(fn, reps):
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


order = os.environ.get("NBX_ENTRY_ORDER", "0")
for cfg in sys.argv[1:]:
    s = systems.make(cfg)
    nb = nbx.Nonbonded(s)
    x = torch.from_numpy(s.x).cuda()
    f = torch.empty_like(x)
    nb.search(x)
    reps = 200 if s.natoms < 200_000 else 20
    r = {"config": cfg, "entry_order": int(order), "natoms": s.natoms}
    r["force_ms"] = timed(lambda: nb.compute(), reps)
    nb.get_f(f)
    r["graph_step_ms"] = timed(lambda: nb.graph_step(x, f, prune=False), reps)
    r["graph_step_prune_ms"] = timed(lambda: nb.graph_step(x, f, prune=True), reps)
    print(json.dumps(r), flush=True)
