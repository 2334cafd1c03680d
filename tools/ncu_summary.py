#!/usr/bin/env python
"""Summarise ncu artefacts into markdown for profiles/.

  python tools/ncu_summary.py launches <launches.csv>        # per-kernel share of an ncu launch list
  python tools/ncu_summary.py report <x.ncu-rep> [label]     # key --set full metrics of one kernel
"""
import collections
import csv
import subprocess
import sys

KEY_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "FMA-heavy (IMAD) pipe active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU issue %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (active)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall: long scoreboard"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall: math pipe throttle"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall: barrier"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall: short scoreboard"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall: not selected"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    idx = {k: i for i, k in enumerate(h)}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) < len(h) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]].split("<")[0].split("(")[0].replace("void ", "").strip().split("::")[-1]
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        ms = {"ns": v / 1e6, "us": v / 1e3, "usecond": v / 1e3, "nsecond": v / 1e6, "ms": v, "msecond": v}.get(unit, v)
        tot[name] += ms
        cnt[name] += 1
    total = sum(tot.values())
    out = ["| kernel | launches | ncu ms (cold, serialised) | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"| `{k}` | {cnt[k]} | {v:.2f} | {100 * v / total:.1f}% |")
    out.append(f"| **total** | {sum(cnt.values())} | {total:.1f} | 100% |")
    return "\n".join(out)


def report(path, label=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
    name = d.get("Kernel Name", ("?", ""))[0].split("(")[0]
    out = [f"**{label or path}** — `{name[:110]}`", "", "| metric | value |", "|---|---|"]
    for key, desc in KEY_METRICS:
        if key in d:
            v, u = d[key]
            out.append(f"| {desc} (`{key}`) | {v} {u} |")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        print(report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""))
