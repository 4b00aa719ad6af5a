"""Row f4 timings: PME (memset + spread + R2C + solve + C2R + gather) and the leap-frog update
per config, CUDA events; parity numbers vs the float64 oracle for the smaller ones.

    python tools/time_pme.py [config ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_01420_b200 import pme, systems  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main(cfg, check):
    s = systems.make(cfg)
    pm = pme.Pme.for_system(s)
    x = torch.from_numpy(s.x).cuda()
    q = torch.from_numpy(s.q).cuda()
    f = torch.zeros_like(x)
    v = torch.zeros_like(x)
    im = torch.ones_like(q)
    r = {"config": cfg, "natoms": s.natoms, "grid": pm.nk}
    r["pme_ms"] = timed(lambda: pm.compute(x, q, out=f), 10)
    r["pme_energy_ms"] = timed(lambda: pm.compute(x, q, out=f, energy=True, virial=True), 3)
    r["leapfrog_ms"] = timed(lambda: pme.leapfrog(x, v, f, im, 0.0), 10)  # dt 0: x, v unchanged
    if check:
        from oracle import pme as P
        fg, (e, vir) = pm.compute(x, q, energy=True, virial=True)
        Eo, fo, vo = P.pme(s.x, s.q, s.box, float(pm_beta(s)), 138.935458, pm.nk, 4)
        fg = fg.cpu().numpy().astype(np.float64)
        r["force_rel_rms"] = float(np.sqrt(((fg - fo) ** 2).sum() / (fo**2).sum()))
        r["energy_rel"] = abs(e - Eo) / abs(Eo)
        r["virial_rel"] = float(np.abs(vir - vo).max() / np.abs(vo).max())
    print(json.dumps(r), flush=True)


def pm_beta(s):
    from paper_2405_01420_b200 import nbx
    return nbx.derive_consts(nbx.make_params(**s.params()))["beta"]


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["rnase24k", "stmv", "water12m"]):
        main(c, check=c in ("rnase24k", "mem82k"))
