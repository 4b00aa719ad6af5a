"""Row f1: feed measured B200 kernel times back into the reference's
own cost-model plug-in point.

The reference prices every NB-path kernel with an affine law per KernelKind
(`CostTable.duration_ns`, /root/reference/pkg/src/mdgpusim/costs.py:137-140) and ingests
measurements through `mdgpusim calibrate --samples timings.cfg`, whose format is
`<kernel>.<index> = <atoms> <duration_ns>` (cli.py:407-433, README.md "calibrate") and whose
fit is `fit_affine` (costs.py:78-107).  This module measures the real sm_100a kernels behind
nbnxm_local, prune_only, pair_search and reduce_forces at several system sizes, writes that
samples file, and restates `fit_affine` so the B200 cost law can be reported without
importing the reference (it is not present on the GPU box).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

KINDS = ("nbnxm_local", "prune_only", "pair_search", "reduce_forces",
         # row f4: the PME stages and the update (pipeline.py:241-257), from nbx_pme_profile
         "grid_memset", "pme_spread", "fft_3d_forward", "pme_solve", "fft_3d_inverse", "pme_gather", "leap_frog")


def fit_affine(points: Sequence[Tuple[int, float]], clamp_floor: bool = True) -> Tuple[float, float]:
    """Restatement of costs.fit_affine (costs.py:78-107): (floor_ns, slope_ns_per_atom)."""
    if len(points) < 2:
        raise ValueError("need at least two samples to fit")
    n = len(points)
    sxx = sum(p[0] * p[0] for p in points)
    sxy = sum(p[0] * p[1] for p in points)
    if n == 2:
        (x1, y1), (x2, y2) = points
        if x1 == x2:
            raise ValueError("all samples at the same atom count")
        slope = (y2 - y1) / (x2 - x1)
        floor = y1 - slope * x1
    else:
        sx = sum(p[0] for p in points)
        sy = sum(p[1] for p in points)
        denom = n * sxx - sx * sx
        if denom == 0:
            raise ValueError("all samples at the same atom count")
        slope = (n * sxy - sx * sy) / denom
        floor = (sy - slope * sx) / n
    if clamp_floor and floor < 0:
        floor = 0.0
        slope = sxy / sxx
    return floor, slope


def samples_to_cfg(samples: Dict[str, List[Tuple[int, float]]], header: str = "") -> str:
    """Render `<kernel>.<i> = <atoms> <duration_ns>` lines (the calibrate input format)."""
    out = [f"# {header}"] if header else []
    for kind in sorted(samples):
        if kind not in KINDS:
            raise ValueError(f"unknown kernel kind {kind!r}")
        for i, (atoms, ns) in enumerate(sorted(samples[kind])):
            out.append(f"{kind}.{i} = {int(atoms)} {float(ns):.1f}")
    return "\n".join(out) + "\n"


def parse_cfg(text: str) -> Dict[str, List[Tuple[int, float]]]:
    """Inverse of samples_to_cfg (mirrors cmd_calibrate's parsing, cli.py:409-421)."""
    by_kind: Dict[str, List[Tuple[int, float]]] = {}
    for line in text.splitlines():
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        key, value = (s.strip() for s in line.split("=", 1))
        kind = key.split(".", 1)[0]
        parts = value.split()
        if len(parts) != 2:
            raise ValueError(f"{key}: expected 'atoms duration_ns'")
        by_kind.setdefault(kind, []).append((int(parts[0].replace("_", "")), float(parts[1])))
    return by_kind


def measure(sizes=(24000, 96000, 384000), reps=20, coulomb="ewald", device=0):
    """Time the NB kernels, the PME stages and the update on water boxes of the given atom
    counts (CUDA events)."""
    import torch

    from . import nbx, systems
    samples: Dict[str, List[Tuple[int, float]]] = {k: [] for k in KINDS}
    for n in sizes:
        s = systems.water_box(n // 3, seed=7, coulomb=coulomb, rc=1.0)
        nb = nbx.Nonbonded(s, device=device)
        x = torch.from_numpy(s.x).cuda(device)
        f = torch.empty_like(x)
        nb.search(x)
        nb.forces(x, out=f)
        st = torch.cuda.current_stream()

        def timed(fn, r=reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            fn()
            torch.cuda.synchronize()
            e0.record(st)
            for _ in range(r):
                fn()
            e1.record(st)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) * 1e6 / r

        samples["nbnxm_local"].append((s.natoms, timed(lambda: nb.compute())))
        samples["prune_only"].append((s.natoms, timed(lambda: nb.prune())))
        samples["reduce_forces"].append((s.natoms, timed(lambda: nb.get_f(f))))
        samples["pair_search"].append((s.natoms, timed(lambda: nb.search(x), r=max(2, reps // 5))))
        nb.close()
        from . import pme
        pm = pme.Pme.for_system(s, device=device)
        q = torch.from_numpy(s.q).cuda(device)
        pm.profile(x, q, out=f)  # warm-up (plans, caches)
        acc = {k: 0.0 for k in pm.STAGES}
        for _ in range(reps):
            for k, v in pm.profile(x, q, out=f).items():
                acc[k] += v
        for k in pm.STAGES:
            samples[k].append((s.natoms, acc[k] * 1e6 / reps))
        v = torch.zeros_like(x)
        im = torch.ones_like(q)
        samples["leap_frog"].append((s.natoms, timed(lambda: pme.leapfrog(x, v, f, im, 0.0))))
    return samples


if __name__ == "__main__":
    import sys
    smp = measure()
    txt = samples_to_cfg(smp, header="B200 sm_100a kernel timings (libnbx), water boxes, Ewald rc=1.0")
    out = sys.argv[1] if len(sys.argv) > 1 else None
    if out:
        open(out, "w").write(txt)
    print(txt)
    for k, pts in smp.items():
        fl, sl = fit_affine(sorted(pts))
        print(f"{k}: floor {fl:.0f} ns, slope {sl:.4f} ns/atom")
