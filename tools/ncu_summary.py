"""Summarise an ncu report (--set full) and/or a launch-list CSV into profiles/ markdown.

    python tools/ncu_summary.py report.ncu-rep out.md [--launches launches.csv] [--title T]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe inst %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe inst %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe inst %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe inst %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe inst %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarize(rep, title):
    hdr, units, rows = raw(rep)
    lines = [f"## {title}", "", f"Source: `{rep}` (ncu --set full --clock-control none)", ""]
    seen = set()
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        if name in seen:
            continue
        seen.add(name)
        lines += [f"### `{name[:110]}`", "", "| metric | value |", "|---|---|"]
        for key, label in METRICS:
            if key in hdr:
                i = hdr.index(key)
                lines.append(f"| {label} (`{key}`) | {r[i]} {units[i]} |")
        st = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), r[i])
              for i, h in enumerate(hdr)
              if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")]
        st = [(k, float(v)) for k, v in st if v and float(v) > 0.05]
        st.sort(key=lambda t: -t[1])
        lines += ["", "Warp stall reasons (per issued instruction): " +
                  ", ".join(f"{k} {v:.2f}" for k, v in st), ""]
    return lines


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = {}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:70]
        v = float(r[vi].replace(",", ""))
        agg.setdefault(name, [0, 0.0])
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = ["## Launch list (gpu__time_duration.sum, cold-cache, serialised)", "",
             f"Source: `{path}`", "", "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda t: -t[1][1]):
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e3:.1f} | {v[1] / 1e3 / v[0]:.1f} | {100 * v[1] / tot:.1f}% |")
    return lines + [""]


if __name__ == "__main__":
    rep, out = sys.argv[1], sys.argv[2]
    title = "ncu summary"
    lines = []
    if "--title" in sys.argv:
        title = sys.argv[sys.argv.index("--title") + 1]
    if rep != "-":
        lines += summarize(rep, title)
    if "--launches" in sys.argv:
        lines += launches(sys.argv[sys.argv.index("--launches") + 1])
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
