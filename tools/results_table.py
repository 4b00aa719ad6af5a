"""Run bench.py (N = 1) on every config and print the BASELINE.md section 4 table rows.

    python tools/results_table.py [--steps K] > gpurun_out/results.md
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = ["water3k", "rnase24k", "rnase24k_lb", "mem82k", "stmv", "stmv_fsw", "stmv_tab", "grappa1.5m", "water12m"]


def main():
    steps = sys.argv[sys.argv.index("--steps") + 1] if "--steps" in sys.argv else "100"
    rows = []
    for c in CONFIGS:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", c, "--steps", steps, "--warmup", "10",
               "--cpu-seconds", "8"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        try:
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            print(f"| {c} | failed: {r.stderr[-300:]!r} |")
            continue
        rows.append(d)
        rf = d["roofline"]
        cpu = d.get("cpu_baseline") or {}
        print(f"| {c} | 1 | {d['value']:.3e} | {d['steps_per_s']:.0f} | {d['ns_per_day']:.1f} | "
              f"{d['kernels_ms']['force_avg']:.3f} | {rf['frac'] * 100:.1f} % useful / {rf['slot_frac'] * 100:.1f} % slots | "
              f"{d['cluster_efficiency']:.2f} | {(cpu.get('value') or 0):.3e} ({cpu.get('cores')} cores) | "
              f"{(d.get('e2e') or {}).get('value', 0):.3e} |", flush=True)
    with open(os.path.join(ROOT, "gpurun_out", "results_rows.json"), "w") as f:
        json.dump(rows, f)


if __name__ == "__main__":
    main()
