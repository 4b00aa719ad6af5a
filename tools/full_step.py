"""Row f4: a GPU-resident MD step of the kernels the reference submits per step for a PME
system (pipeline.py:222-257) minus the ones out of scope (listed forces, constraints):
NB path with its cadence (X op, prune every 10, search every 100, force, F op) + PME
(memset, spread, R2C, solve, C2R, gather) + leap-frog update.  CUDA events over K steps.

dt = 0 in the update: with no bonded forces or constraints the molecules would fly apart, so
positions are kept fixed; the update kernel still runs at full cost.  The result is an upper
bound on the application rate (no listed forces, constraints or PME-PP communication).

    python tools/full_step.py [config ...] [--steps K] [--graphs]

--graphs replays each non-search step as one CUDA graph (Nonbonded.md_step, nbx_step_graph_pme).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01420_b200 import nbx, pme, systems  # noqa: E402


def run(cfg, steps, grid_order=True, graphs=False):
    s = systems.make(cfg)
    nb = nbx.Nonbonded(s)
    pm = pme.Pme.for_system(s)
    x = torch.from_numpy(s.x).cuda()
    q = torch.from_numpy(s.q).cuda()
    f = torch.empty_like(x)
    v = torch.zeros_like(x)
    im = torch.ones_like(q)
    st = torch.cuda.current_stream()

    def one(k):
        if graphs:  # non-search steps as one graph launch (nbx_step_graph_pme)
            nb.md_step(x, f, v, im, 0.0, k, pm, graphs=True)
            return
        if grid_order:  # PME on the NB grid's cluster-ordered atoms, forces via the F op
            nb.step(x, f, k, pme=pm)
        else:
            nb.step(x, f, k)
            pm.compute(x, q, out=f)
        pme.leapfrog(x, v, f, im, 0.0)

    for k in range(10):
        one(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(10, 10 + steps):
        one(k)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    out = {"config": cfg, "natoms": s.natoms, "steps": steps, "ms_per_step": ms, "pme_on_nb_grid": grid_order, "graphs": graphs,
           "ns_per_day_upper_bound": 86.4 * s.dt_fs / ms if hasattr(s, "dt_fs") else 86.4 * 2.0 / ms,
           "pme_grid": pm.nk, "gpu_launches_nb_pme": nb.launch_count() + pm.launch_count()}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    steps = 100
    if "--steps" in args:
        i = args.index("--steps")
        steps = int(args[i + 1])
        del args[i:i + 2]
    user_order = "--user-order" in args
    graphs = "--graphs" in args
    args = [a for a in args if a not in ("--user-order", "--graphs")]
    for c in (args or ["stmv", "water12m"]):
        run(c, steps, grid_order=not user_order, graphs=graphs)
