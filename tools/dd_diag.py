"""Diagnose a DD-vs-single-GPU force mismatch from tests/dd_gpu_worker.py output: the atoms with
the largest |df| / rms|f|, their force magnitudes and nearest-neighbour distances.

    python tools/dd_diag.py <out.npz> <config> [key]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2405_01420_b200 import systems  # noqa: E402

out, cfg = sys.argv[1], sys.argv[2]
key = sys.argv[3] if len(sys.argv) > 3 else "f4"
d = np.load(out)
f, fr = d[key], d[key + "_ref"]
rms = np.sqrt((fr ** 2).sum(1).mean())
df = np.sqrt(((f - fr) ** 2).sum(1))
top = np.argsort(df)[::-1][:10]
s = systems.make(cfg)
rng = np.random.default_rng(3)
disp = rng.uniform(-0.01, 0.01, size=s.x.shape).astype(np.float32)
rng2 = np.random.default_rng(4)
disp2 = rng2.uniform(-0.015, 0.015, size=s.x.shape).astype(np.float32)
x = (s.x + disp + disp2).astype(np.float64) if key == "f4" else (s.x + disp).astype(np.float64)
box = s.box.astype(np.float64)
print("rms |f|", rms, "rel rms", np.sqrt(((f - fr) ** 2).sum() / (fr ** 2).sum()))
for a in top:
    dx = x - x[a]
    dx -= box * np.round(dx / box)
    r = np.sqrt((dx * dx).sum(1))
    r[a] = 1e9
    nn = np.argsort(r)[:3]
    print(f"atom {a} |df|/rms {df[a] / rms:.3e} |f_ref| {np.linalg.norm(fr[a]):.4g} |f| {np.linalg.norm(f[a]):.4g} "
          f"x {x[a]} nn {[(int(b), round(float(r[b]), 4)) for b in nn]} wrapped {x[a] % box}")
