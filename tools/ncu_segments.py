#!/usr/bin/env python
"""Per-phase breakdown of one kernel from an ncu report: the SASS is cut at
BAR/EXIT instructions (one segment per NTT round for the block kernels) and
each segment's warp-stall samples, executed instructions, FP64 share and
shared/global memory instruction counts are printed.
Usage: ncu_segments.py report.ncu-rep [launch_index]"""
import csv
import io
import re
import subprocess
import sys

R = ["stall_barrier", "stall_long_sb", "stall_short_sb", "stall_wait", "stall_math", "stall_mio",
     "stall_not_selected", "stall_selected", "stall_lg", "stall_dispatch", "stall_branch_resolving", "stall_no_inst"]


def main(path, launch=0):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(launch), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    data, seen = [], set()
    for r in rows[2:]:
        if len(r) != len(h) or r[0] == "Address" or r[0] in seen:
            continue
        seen.add(r[0])
        data.append(r)

    def f(r, k):
        try:
            return float(r[ix[k]] or 0)
        except (KeyError, ValueError):
            return 0.0

    def new(a):
        return {"s": 0, "inst": 0, "fp64": 0, "lds": 0, "sts": 0, "ldg": 0, "start": a, "r": dict.fromkeys(R, 0)}
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
    segs, cur = [], new(data[0][0])
    for r in data:
        op = re.sub(r"^@!?U?P\w+\s+", "", r[ix["Source"]].strip()).split(" ")[0]
        cur["s"] += f(r, "Warp Stall Sampling (All Samples)")
        ie = f(r, "Instructions Executed")
        cur["inst"] += ie
        cur["fp64"] += ie if op.startswith(("DADD", "DMUL", "DFMA")) else 0
        cur["lds"] += ie if op.startswith("LDS") else 0
        cur["sts"] += ie if op.startswith("STS") else 0
        cur["ldg"] += ie if op.startswith("LDG") else 0
        for k in R:
            cur["r"][k] += f(r, k)
        if op.startswith(("BAR", "EXIT")):
            cur["end"] = r[0]
            segs.append(cur)
            cur = new(r[0])
    segs.append(cur)
    ti = sum(s["inst"] for s in segs)
    print(f"{len(data)} SASS lines, {ti:.3g} warp instructions, FP64 share {sum(s['fp64'] for s in segs) / ti:.2f}")
    for s in segs:
        if s["s"] / tot < 0.01:
            continue
        top = sorted(s["r"].items(), key=lambda kv: -kv[1])[:4]
        print(f"{s['start'][-5:]}-{s.get('end', 'end')[-5:]} time {100 * s['s'] / tot:5.1f}% inst {100 * s['inst'] / ti:5.1f}% "
              f"fp64/inst {s['fp64'] / max(s['inst'], 1):.2f} lds {s['lds'] / 1e6:.1f}M sts {s['sts'] / 1e6:.1f}M "
              f"ldg {s['ldg'] / 1e6:.1f}M | " + ", ".join(f"{k[6:]} {100 * v / max(s['s'], 1):.0f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
