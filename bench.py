#!/usr/bin/env python
"""bench.py -- NB-path MD steps of the B200-native NBNXM engine (libnbx.so).

Metric (BASELINE.json): nonbonded pair-interactions/s and MD steps/s (ns/day) at 1/2/4/8
B200 vs the FP32 roofline.  One "step" is one NB-path MD step with the reference cadence
(pipeline.py:222-235): X buffer op + force kernel + F buffer op every step, the rolling
prune every prune_every (10) steps, grid + pair search every nstlist (100) steps.  A step
evaluates every in-cut-off pair once, so pair-interactions/s = pairs_per_step * steps / s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config water12m] [--impl nbx|reference]

N = 1: single domain on cuda:0.  N > 1 (torchrun, one rank per GPU): spatial domain
decomposition (paper_2405_01420_b200.dd) with NCCL halo exchange; strong scaling (the box is
fixed).  `--impl reference` times the CPU implementation of the path (the C oracle port,
all host threads, rank 0 only) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "nonbonded pair-interactions/s and MD steps/s (ns/day) at 1/2/4/8 B200 vs FP32 roofline"
UNIT = "pair-interactions/s"
# Algorithmic FP32 flops per in-cut-off pair of the force-only kernel, counted once from
# pairmath.cuh / force.cu (FADD/FMUL/MUFU = 1, FFMA = 2) and frozen.
FLOPS_PER_PAIR = {"ewald": 57, "rf": 33, "ewald-tab": 43}
# ... and as the shipped F-only tile issues them (pairmath.cuh ewald_coul_r2 + force.cu tile():
# 3 (dx, dy, dz) + 5 (r2) + 1 MUFU.RSQ + 3 (r^-2, r^-3, r^-6) + 3 (LJ) + 22 (rational: FADD2,
# 4 FFMA2, MUFU.RCP, FMUL, FFMA) + 1 (qq) + 1 (Coulomb) + 2 (fscal) + 12 (i and j forces) = 53)
FLOPS_ISSUED = {"ewald": 53}
# combination-rule LJ adds the per-pair parameter arithmetic (nbx.h NBX_LJ_COMB_*)
LJ_EXTRA_FLOPS = {"comb-geom": 2, "comb-lb": 8}
DESC = {
    "water3k": "SPC/E water box 3k atoms (1k waters), reaction-field, rc=0.9 nm",
    "rnase24k": "RNase-sized 24,024-atom solvated protein-like box, Ewald real-space, rc=1.0 nm",
    "mem82k": "benchMEM-sized 82k-atom membrane-like box, LJ + Ewald, dynamic pruning every 10 steps",
    "stmv": "STMV-sized 1,066,628-atom water/protein box, Ewald, rc=1.2 nm",
    "stmv_fsw": "STMV-sized box with force-switch LJ (rvdw_switch 1.0 nm, rc 1.2 nm), Ewald",
    "stmv_tab": "STMV-sized box, the paper's STMV kernel flavour: tabulated Ewald + force-switch LJ, rc 1.2 nm",
    "water12m": "12M-atom water box, Ewald, rc=1.0 nm (strong-scaling sweep 1/2/4/8)",
    "rnase24k_lb": "RNase-sized 24,024-atom protein-like box, Ewald, Lorentz-Berthelot combination-rule LJ",
    "rnase24k_geom": "RNase-sized 24,024-atom protein-like box, Ewald, geometric combination-rule LJ",
    "grappa1.5m": "Grappa kernel flavour (tabulated Ewald + LB combination-rule LJ), 1.5M-atom uniform water box, rc=1.0 nm",
}
L2_BYTES = 126 * 1024 * 1024
NATOMS = {"water3k": 3000, "rnase24k": 24024, "mem82k": 82000, "stmv": 1066628, "stmv_fsw": 1066628,
          "stmv_tab": 1066628,
          "water12m": 12_000_000, "rnase24k_lb": 24024, "rnase24k_geom": 24024, "grappa1.5m": 1_500_000}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="water12m", choices=sorted(DESC))
    ap.add_argument("--impl", default="nbx", choices=["nbx", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bounded CPU baseline budget")
    return ap.parse_args()


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, interval_ms=100, enabled=True):
        self.index = index
        self.interval_ms = int(interval_ms)
        self.enabled = enabled
        self.proc = None
        self.f = None

    def start(self):
        if not self.enabled:
            return self
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", str(self.interval_ms)], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return self
        # nvidia-smi's NVML start-up contends with this process's CUDA calls for a fraction of a
        # second: wait for its first sample so the start-up never lands in a timed region
        t0 = time.time()
        while time.time() - t0 < 5.0:
            self.f.flush()
            if os.path.getsize(self.f.name) > 0:
                break
            time.sleep(0.05)
        time.sleep(0.3)
        return self

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        clocks, maxc, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                clocks.append(float(r[1]))
                maxc.append(float(r[2]))
                power.append(float(r[3]))
                for k, nm in enumerate(names):
                    if r[5 + k].strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if clocks:
            busy = sorted(c for c in clocks if c > 0.5 * max(clocks)) or sorted(clocks)
            out = {"sm_mhz": busy[len(busy) // 2], "sm_max_mhz": max(maxc), "reasons": sorted(reasons),
                   "samples": len(clocks), "power_w_max": max(power) if power else None}
        return out


# ------------------------------------------------------------------------------ helpers
def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def load_traffic(config, n):
    """dram bytes per force launch from the committed ncu --set full capture, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(f"{config}:{n}")
    except Exception:
        return None


def cpu_sample_system(config):
    """A bounded sample of the workload for the CPU port: same generator/parameters, fewer atoms."""
    from paper_2405_01420_b200 import systems
    n = {"water3k": None, "rnase24k": None, "mem82k": 24000, "stmv": 48000, "stmv_fsw": 48000, "stmv_tab": 48000,
         "water12m": 48000, "rnase24k_lb": None, "rnase24k_geom": None, "grappa1.5m": 48000}[config]
    return systems.make(config, n), n


def time_cpu_port(config, budget_s, steps=None, warmup=0):
    """Oracle port (C, OpenMP, all host threads) on the bounded sample, with the GPU arm's
    cadence and era composition: step k searches (grid + search + prune) when k % nstlist == 0,
    prunes when k % prune_every == 0, and otherwise runs the X op; every step runs the force
    evaluation and the F op.  pairs/s = in-cut-off pairs / era-composed step time."""
    from oracle import oracle as O
    s, n = cpu_sample_system(config)
    on = O.OracleNonbonded(s)
    on.search(s.x)
    pairs = on.count_pairs()
    cores = len(os.sched_getaffinity(0))
    on.forces(flags=0)  # warm the thread pool / caches
    for k in range(warmup):
        on.put_x(s.x)
        on.forces(flags=0)
    t0 = time.perf_counter()
    times, kinds = [], []
    k = 0
    while True:
        kind = step_kind(k, s.nstlist, s.prune_every)
        t = time.perf_counter()
        if kind == "search":
            on.search(s.x)
        else:
            on.put_x(s.x)
            if kind == "prune":
                on.prune()
        on.forces(flags=0)
        times.append(time.perf_counter() - t)
        kinds.append(kind)
        k += 1
        if steps is not None and k >= steps:
            break
        # budget mode: at least one prune step (k > prune_every) before stopping
        if steps is None and (time.perf_counter() - t0) >= budget_s and k > s.prune_every:
            break
    era_s, by_kind, counts = compose_era(times, kinds, s.nstlist, s.prune_every)
    sample = (f"scalar C oracle (the correctness restatement: -ffp-contract=off, AoS, no SIMD kernel -- not "
              f"a tuned CPU NBNXM), OpenMP over {cores} threads, on a {s.natoms}-atom sample box of the same "
              f"generator and parameters ({k} NB-path steps with the reference cadence: search every "
              f"{s.nstlist}, prune every {s.prune_every}, X op / force / F op every step; era-composed as "
              f"on the GPU; {pairs} pairs per step; static coordinates)")
    return {"value": pairs / era_s, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
            "ms_per_eval": 1e3 * era_s, "ms_by_kind": {kk: round(1e3 * v, 3) for kk, v in by_kind.items()},
            "kind_counts": counts, "pairs_per_eval": pairs, "reps": k}


# ------------------------------------------------------------------------------ cadence
def step_kind(step, nstlist, prune_every):
    """'search' | 'prune' | 'plain' by the reference cadence (pipeline.py:222-235)."""
    if step % nstlist == 0:
        return "search"
    if prune_every and step % prune_every == 0:
        return "prune"
    return "plain"


def compose_era(step_ms, kinds, nstlist, prune_every):
    """Mean ms per step over one nstlist era from the per-kind means measured in the window:
    (t_search + n_prune t_prune + n_plain t_plain) / nstlist with the cadence's counts
    (1 search, nstlist/prune_every - 1 prunes, the rest plain).  A window that starts with a
    search step and holds >= prune_every + 1 steps measures all three kinds, so a short K
    weighs the search step exactly as a full era does (no search-free windows)."""
    by = {}
    for t, k in zip(step_ms, kinds):
        by.setdefault(k, []).append(t)
    mean = {k: sum(v) / len(v) for k, v in by.items()}
    t_plain = mean.get("plain", mean.get("prune", 0.0))
    t_prune = mean.get("prune", t_plain)
    t_search = mean.get("search", t_prune)
    n_prune = (nstlist // prune_every - 1) if prune_every else 0
    n_plain = nstlist - 1 - n_prune
    era = (t_search + n_prune * t_prune + n_plain * t_plain) / nstlist
    return era, {k: round(v, 4) for k, v in mean.items()}, {k: len(v) for k, v in by.items()}


# MD-like motion between steps: x += v dt with per-atom velocities of fixed
# magnitude, reversed every nstlist steps so atoms oscillate about their start.  The rms
# displacement over one nstlist era (~0.05 nm) matches liquid-water self-diffusion over the
# era's 0.2 ps (D = 2.3e-9 m^2/s: sqrt(6 D t) = 0.05 nm); lists stay valid within the
# 0.1 nm Verlet buffer, pruning and searching see moving coordinates.
ERA_RMS_DISP_NM = 0.05


def motion_sign(step, nstlist):
    """+1 on the steps of even eras, -1 on odd ones (step k moves by sign(k) v dt)."""
    return 1.0 if ((step - 1) // nstlist) % 2 == 0 else -1.0


def motion_velocities(n, nstlist, dt_ps, seed=11):
    import numpy as np
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(n, 3)).astype(np.float32)
    v *= ERA_RMS_DISP_NM / (np.sqrt(3.0) * nstlist * dt_ps)
    return v


# ------------------------------------------------------------------------------ nbx arm, N = 1
def run_single(args):
    import numpy as np
    import torch

    from paper_2405_01420_b200 import nbx, pme, systems

    torch.cuda.set_device(0)
    s = systems.make(args.config)
    nb = nbx.Nonbonded(s, device=0)
    x = torch.from_numpy(s.x).cuda()
    f = torch.empty_like(x)
    st = torch.cuda.current_stream()
    peak = nb.fma_peak_tflops()
    dt_ps = s.dt_fs * 1e-3
    vel = torch.from_numpy(motion_velocities(s.natoms, s.nstlist, dt_ps)).cuda()
    zero_im = torch.zeros(s.natoms, dtype=torch.float32, device="cuda")  # inv_mass 0: v is kept
    zero_f = torch.zeros_like(x)  # the update's force input (0 * f would still carry a NaN)

    def move(xx, step):
        # x += sign(step) v dt (HBM-bound, between the step events)
        pme.leapfrog(xx, vel, zero_f, zero_im, motion_sign(step, s.nstlist) * dt_ps)

    # small boxes are launch-bound: replay non-search steps as CUDA graphs
    graphs = s.natoms < 500_000
    # setup search, then W warm-up steps numbered nstlist-W .. nstlist-1 (they include prune
    # steps), so the timed window starts with the era's search step
    nb.step(x, f, 0, graphs=graphs)
    # a second search after motion: the search's single-pass buffers are sized by the first, so
    # from here on steps allocate nothing (device_allocs_in_timed_region)
    move(x, 1)
    nb.step(x, f, 0, graphs=graphs)
    for k in range(args.warmup):
        step = max(1, s.nstlist - args.warmup + k)
        move(x, step)
        nb.step(x, f, step, graphs=graphs)
    if graphs:  # instantiate both step graphs before the timed region
        nb.graph_step(x, f, prune=True)
        nb.graph_step(x, f, prune=False)
    torch.cuda.synchronize()
    sizes = nb.list_sizes()
    nslots = nb.grid_info()["nslots"]
    working = nslots * 16 * 3 + sizes["n_cj_outer"] * 16 + sizes["n_pool"] * 64
    flush = working < 2 * L2_BYTES
    scratch = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda") if flush else None

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    evf = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(0, interval_ms=250).start()  # NVML polls contend with CUDA calls
    torch.cuda.synchronize()
    l0 = nb.launch_count()
    a0 = nb.alloc_count()
    kinds = [step_kind(k, s.nstlist, s.prune_every) for k in range(K)]
    pairs0 = None
    w0.record(st)
    for k in range(K):
        if k:
            move(x, k)
        if flush:
            scratch.fill_(float(k))
        ev[k][0].record(st)
        if graphs and kinds[k] != "search":
            nb.graph_step(x, f, prune=kinds[k] == "prune")
        else:
            if kinds[k] == "search":
                nb.search(x)
            else:
                nb.put_x(x)
                if kinds[k] == "prune":
                    nb.prune()
            evf[k][0].record(st)
            nb.compute()
            evf[k][1].record(st)
            nb.get_f(f)
        ev[k][1].record(st)
    w1.record(st)
    torch.cuda.synchronize()
    launches = nb.launch_count() - l0 + (K - 1)  # + the K - 1 motion updates (nbx_leapfrog)
    allocs = nb.alloc_count() - a0
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    era_ms, kind_ms, kind_n = compose_era(step_ms, kinds, s.nstlist, s.prune_every)
    window_ms = w0.elapsed_time(w1)
    # in-cut-off pairs per step: the inner list at the window's end, and the list a search of
    # the window's first coordinates builds (replayed below); the motion changes them < 0.1 %
    pairs_end, slots_end = nb.count_pairs()
    if graphs:  # force kernel alone, back to back on the same stream
        for k in range(K):
            evf[k][0].record(st)
            nb.compute()
            evf[k][1].record(st)
        nb.get_f(f)  # clears the cluster force buffer again
        torch.cuda.synchronize()
    force_ms = [evf[k][0].elapsed_time(evf[k][1]) for k in range(K)]
    xs = torch.from_numpy(s.x).cuda()
    nb.search(xs)  # the window's first list (same x as its search step up to the warm-up motion)
    pairs_start, slots_start = nb.count_pairs()
    pairs = 0.5 * (pairs_start + pairs_end)
    slots = 0.5 * (slots_start + slots_end)
    ms_per_step = era_ms
    value = pairs / (ms_per_step * 1e-3)
    t_force = sum(force_ms) / len(force_ms)
    fl = FLOPS_PER_PAIR[s.coulomb] + LJ_EXTRA_FLOPS.get(s.lj_modifier, 0)
    fl_iss = FLOPS_ISSUED.get(s.coulomb, fl) + LJ_EXTRA_FLOPS.get(s.lj_modifier, 0)
    achieved = pairs * fl / (t_force * 1e-3) / 1e12
    achieved_iss = pairs * fl_iss / (t_force * 1e-3) / 1e12
    slot_tf = slots * fl / (t_force * 1e-3) / 1e12

    # e2e: the public API with host buffers -- every step copies x from pinned host memory
    # (H2D) and reads f back (D2H) inside the timed region; same cadence and era composition
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(s.x.copy()).pin_memory()
        fh = torch.empty((s.natoms, 3), dtype=torch.float32).pin_memory()
        xd = torch.empty_like(x)
        Ke = max(1, min(K, 50))
        eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(Ke)]
        ekinds = [step_kind(k, s.nstlist, s.prune_every) for k in range(Ke)]
        torch.cuda.synchronize()
        for k in range(Ke):
            eev[k][0].record(st)
            xd.copy_(xh, non_blocking=True)
            nb.step(xd, f, k, graphs=graphs)
            fh.copy_(f, non_blocking=True)
            eev[k][1].record(st)
        torch.cuda.synchronize()
        ems = [a.elapsed_time(b) for a, b in eev]
        e_era, e_kind_ms, _ = compose_era(ems, ekinds, s.nstlist, s.prune_every)
        e2e = {"value": pairs / (e_era * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(xh.numel() * 4),
               "d2h_bytes_per_step": int(fh.numel() * 4), "steps": Ke, "ms_per_step": e_era,
               "ms_per_step_by_kind": e_kind_ms, "window_ms_per_step": sum(ems) / Ke,
               "api": "paper_2405_01420_b200.nbx.Nonbonded.step (ctypes -> libnbx.so C-ABI)"}

    cpu = None
    if not args.no_cpu_baseline:
        try:
            cpu = time_cpu_port(args.config, args.cpu_seconds)
        except Exception as e:  # reported, never substituted
            cpu = {"value": None, "error": str(e)[:200]}

    traffic = load_traffic(args.config, 1)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {DESC[args.config]}", "natoms": s.natoms,
                   "nstlist": s.nstlist, "prune_every": s.prune_every, "rc": s.rc,
                   "rlist_outer": s.rlist_outer, "rlist_inner": s.rlist_inner,
                   "parallelism": "single domain",
                   "l2": ("L2 flushed (2x126 MB write) before every timed step" if flush
                          else f"inputs larger than L2 (xyzq+lists {working / 2**20:.0f} MiB)"),
                   "motion": (f"x += v dt between steps (v reversed every nstlist steps; {ERA_RMS_DISP_NM} nm rms "
                              "per era), outside the step events"),
                   "step_time": ("one nstlist era composed from the window's per-kind step means: (t_search + "
                                 f"{s.nstlist // s.prune_every - 1} t_prune + "
                                 f"{s.nstlist - s.nstlist // s.prune_every} t_plain) / {s.nstlist}; the window "
                                 "starts with a search step")},
        "steps_per_s": 1e3 / ms_per_step,
        "ns_per_day": 86.4 * s.dt_fs / ms_per_step,
        "pairs_per_step": pairs,
        "pair_slots_per_step": slots,
        "cluster_efficiency": pairs / slots if slots else None,
        "step_ms": {"era": era_ms, "window_mean": sum(step_ms) / K, "window_incl_motion": window_ms / K,
                    "by_kind": kind_ms, "kind_counts": kind_n, "median": sorted(step_ms)[K // 2], "max": max(step_ms)},
        "kernels_ms": {"force_avg": t_force},
        "roofline": {"bound": "fp32", "kernel": "k_force (NBNXM force, F only)", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": "measured on this GPU: register-resident FFMA loop (nbx_fma_peak)",
                     "flops_per_pair": fl, "flops_per_pair_note": "frozen before optimisation (DESIGN.md section 5)",
                     "flops_per_pair_issued": fl_iss, "achieved_issued": achieved_iss, "frac_issued": achieved_iss / peak,
                     "slot_tflops": slot_tf, "slot_frac": slot_tf / peak},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "device_allocs_in_timed_region": int(allocs),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    # all the host threads: torchrun (N > 1) exports OMP_NUM_THREADS=1 to every rank; the oracle's
    # OpenMP runtime reads the variable when it is first loaded, which happens below
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    t0 = time.perf_counter()
    r = time_cpu_port(args.config, None, steps=args.steps, warmup=args.warmup)
    wall = time.perf_counter() - t0
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_eval"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {DESC[args.config]}", "natoms": NATOMS[args.config],
                   "nstlist": 100, "prune_every": 10,
                   "parallelism": "host CPU (the reference path has no GPU implementation)"},
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "port",
                         "sample": r["sample"]},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("the reference (mdgpusim) computes no forces (SPEC.md:8); this arm times the CPU "
                 "restatement of the path (oracle/nbx_oracle.c: a scalar correctness oracle, not a tuned "
                 "SIMD CPU NBNXM) on the box's host cores, on a 48k-atom sample box, with the GPU arm's step "
                 "cadence (search / prune / X op / force / F op) and era composition: a stated baseline"),
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


def _json_only_stdout():
    """Keep stdout for the JSON line alone: native libraries that write to fd 1 (NCCL's
    version banner under NCCL_DEBUG, cuFFT/driver notices) are sent to stderr, Python's
    sys.stdout keeps the original descriptor."""
    try:
        sys.stdout.flush()
        keep = os.dup(1)
        os.dup2(2, 1)
        sys.stdout = os.fdopen(keep, "w", buffering=1)
    except OSError:
        pass


def main():
    args = parse()
    _json_only_stdout()
    # no cyclic-GC pauses inside timed regions (a gen-2 pass during a Python-side search /
    # repartition step stalls the GPU that step waits on); reference counting still frees
    gc.collect()
    gc.disable()
    if args.impl == "reference":
        run_reference(args)
        return
    rank, world, local = dist_env()
    if world > 1 or args.gpus > 1:
        from paper_2405_01420_b200 import dd
        dd.bench(args, METRIC, UNIT, FLOPS_PER_PAIR, DESC, ClockSampler, time_cpu_port, load_traffic,
                 step_kind=step_kind, compose_era=compose_era, motion_velocities=motion_velocities,
                 motion_sign=motion_sign)
        return
    run_single(args)


if __name__ == "__main__":
    main()
