"""Per-phase CUDA-event timings of the NB path for one config (the bench's breakdown).

    python tools/time_kernels.py [config ...]
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
    fn()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main(cfg):
    s = systems.make(cfg)
    nb = nbx.Nonbonded(s)
    x = torch.from_numpy(s.x).cuda()
    f = torch.empty_like(x)
    nb.search(x)
    r = {"config": cfg, "natoms": s.natoms}
    r["search_ms"] = timed(lambda: nb.search(x), 3)
    r["prune_ms"] = timed(lambda: nb.prune(), 10)
    r["put_x_ms"] = timed(lambda: nb.put_x(x), 20)
    r["force_ms"] = timed(lambda: nb.compute(), 10)
    r["force_virial_ms"] = timed(lambda: nb.compute(virial=True), 5)
    r["force_energy_ms"] = timed(lambda: nb.compute(energy=True, virial=True), 5)
    r["get_f_ms"] = timed(lambda: nb.get_f(f), 20)
    p, sl = nb.count_pairs()
    r.update(nb.list_sizes())
    r["pairs"] = p
    r["slots"] = sl
    r["step_ms_model"] = r["put_x_ms"] + r["force_ms"] + r["get_f_ms"] + r["prune_ms"] / s.prune_every + \
        r["search_ms"] / s.nstlist
    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["stmv"]):
        main(c)
