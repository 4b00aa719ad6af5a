"""Build force-kernel variants (-D flags) and time them on a GPU.

    python tools/force_variants.py build            # here (nvcc cross-compile)
    python tools/force_variants.py run [config]     # on the GPU box
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "scratch", "variants")
VARIANTS = {
    "base": [],
    "g2": ["-DNBX_VF_G=2"],  # energy kernels: the force's G(z) reciprocal without the Newton step
}
# sources whose objects depend on the -D flags (the rest are built once and shared)
FLAG_SOURCES = ("force.cu", "search.cu")


def build():
    sys.path.insert(0, ROOT)
    from paper_2405_01420_b200 import build as B
    os.makedirs(OUT, exist_ok=True)
    shared = {}
    for name, flags in VARIANTS.items():
        objs = []
        for src in B.SOURCES:
            if src not in FLAG_SOURCES and src in shared:
                objs.append(shared[src])
                continue
            o = os.path.join(OUT, f"{name}_{src}.o")
            extra = B.PER_FILE.get(src, [])
            cmd = [B._nvcc(), *B.ARCH, *B.NVCC_FLAGS, *extra, *flags, "-c", os.path.join(B.CSRC, src), "-o", o]
            subprocess.check_call(cmd, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            objs.append(o)
            if src not in FLAG_SOURCES:
                shared[src] = o
        subprocess.check_call([B._nvcc(), *B.ARCH, "-shared", "-o", os.path.join(OUT, f"libnbx_{name}.so"), *objs,
                               "-lcudart", "-lcufft"])
        print("built", name, flush=True)


def run_one(name, cfg, reps=20):
    os.environ["NBX_LIB"] = os.path.join(OUT, f"libnbx_{name}.so")
    sys.path.insert(0, ROOT)
    import torch
    from paper_2405_01420_b200 import nbx, systems
    cname, _, n = cfg.partition(":")
    s = systems.make(cname, int(n) if n else None)
    nb = nbx.Nonbonded(s)
    x = torch.from_numpy(s.x).cuda()
    f = torch.empty_like(x)
    nb.search(x)
    nb.forces(x, out=f)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if os.environ.get("NBX_VARIANT_FLUSH") == "1":
        # cold L2 before every launch, as bench.py does for inputs smaller than 2x L2
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
        tot = 0.0
        for _ in range(reps):
            flush.fill_(1.0)
            e0.record(st)
            nb.compute()
            e1.record(st)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        ms = tot / reps
    else:
        e0.record(st)
        for _ in range(reps):
            nb.compute()
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
    f.zero_()
    nb.forces(x, out=f)
    torch.cuda.synchronize()
    p, sl = nb.count_pairs()
    tag = name + ("_packed" if os.environ.get("NBX_PACKED_FORCE") == "1" else "")
    import numpy as np
    fn = f.cpu().numpy().astype(np.float64)
    np.save(os.path.join(OUT, f"f_{tag}_{cfg}.npy"), fn)
    e0.record(st)
    for _ in range(reps):
        nb.prune()
    e1.record(st)
    torch.cuda.synchronize()
    prune_ms = e0.elapsed_time(e1) / reps
    e0.record(st)
    for _ in range(3):
        nb.search(x)
    e1.record(st)
    torch.cuda.synchronize()
    search_ms = e0.elapsed_time(e1) / 3
    e0.record(st)
    for _ in range(3):
        nb.compute(energy=True, virial=True)
    e1.record(st)
    torch.cuda.synchronize()
    vf_ms = e0.elapsed_time(e1) / 3
    out = {"variant": tag, "config": cfg, "force_ms": ms, "prune_ms": prune_ms, "search_ms": search_ms, "vf_ms": vf_ms, "slot_tflops": sl * 57 / ms / 1e9,
           "pairs_per_s": p / ms * 1e3}
    ref = os.path.join(OUT, f"f_base_{cfg}.npy")
    if os.path.exists(ref) and tag != "base":
        fr = np.load(ref)
        out["rel_rms_vs_base"] = float(np.sqrt(((fn - fr) ** 2).sum() / (fr ** 2).sum()))
    return out


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    elif sys.argv[1] == "run":
        cfg = sys.argv[2] if len(sys.argv) > 2 else "stmv"
        names = sys.argv[3].split(",") if len(sys.argv) > 3 else list(VARIANTS)
        for n in names:
            r = subprocess.run([sys.executable, __file__, "one", cfg, n], capture_output=True, text=True)
            print(r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:], flush=True)
    elif sys.argv[1] == "one":
        print(json.dumps(run_one(sys.argv[3], sys.argv[2])))
