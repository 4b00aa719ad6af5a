"""Energy-kernel accuracy against the oracle for one libnbx build (NBX_LIB selects a variant).

    python tools/vf_accuracy.py oracle            # oracle energies / virial -> scratch/vf_ref_*.npz
    NBX_LIB=... python tools/vf_accuracy.py gpu   # GPU VF step vs those, one JSON line per case

Cases: the configs test_gpu_parity checks at energy steps, plus water3k after a random motion
(the prune-after-motion case).  Prints relative energy errors, the virial error (max-normalised)
and the force errors; the bars are 1e-6 / 1e-6 / 1e-5 RMS (tests/helpers.py).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_01420_b200 import systems  # noqa: E402
from tests.helpers import force_errors  # noqa: E402

CASES = ["water3k", "water3k:moved", "rnase24k", "mem82k", "rnase24k_lb", "rnase24k_geom", "stmv"]
OUT = os.path.join(ROOT, "scratch")


def case_x(name):
    base, _, mod = name.partition(":")
    s = systems.make(base)
    x = s.x
    if mod == "moved":
        rng = np.random.default_rng(7)
        x = (s.x + rng.uniform(-0.03, 0.03, size=s.x.shape)).astype(np.float32)
    return s, x


def oracle():
    from oracle import oracle as O
    os.makedirs(OUT, exist_ok=True)
    for c in CASES:
        s, x = case_x(c)
        on = O.OracleNonbonded(s)
        on.search(x)
        fo, eo, viro, _ = on.forces()
        np.savez(os.path.join(OUT, f"vf_ref_{c.replace(':', '_')}.npz"), f=fo, e=eo, vir=viro)
        print("oracle", c, flush=True)


def gpu():
    import torch
    from paper_2405_01420_b200 import nbx
    for c in CASES:
        s, x = case_x(c)
        r = np.load(os.path.join(OUT, f"vf_ref_{c.replace(':', '_')}.npz"))
        nb = nbx.Nonbonded(s, device=0)
        xd = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
        nb.search(xd)
        f, (e, vir) = nb.forces(xd, energy=True, virial=True)
        torch.cuda.synchronize()
        e = np.asarray(e, np.float64)
        erel = (np.abs(e - r["e"]) / np.abs(r["e"])).tolist()
        vrel = float(np.abs(np.asarray(vir) - r["vir"]).max() / np.abs(r["vir"]).max())
        frms, fmax = force_errors(f.cpu().numpy().astype(np.float64), r["f"])
        ok = bool(max(erel) <= 1e-6 and vrel <= 1e-6 and frms <= 1e-5 and fmax <= 1e-4)
        print(json.dumps({"lib": os.path.basename(os.environ.get("NBX_LIB", "libnbx.so")), "case": c,
                          "e_rel": erel, "vir_rel": vrel, "f_rms": float(frms), "f_max": float(fmax), "ok": ok}), flush=True)


if __name__ == "__main__":
    {"oracle": oracle, "gpu": gpu}[sys.argv[1]]()
