#!/usr/bin/env python
"""Per-opcode / per-reason warp-stall breakdown of one kernel from an ncu report
(`ncu -i X --page source --csv --print-source sass`). Usage: ncu_stalls.py rep"""
import collections
import csv
import io
import re
import subprocess
import sys

REASONS = ["stall_barrier", "stall_long_sb", "stall_short_sb", "stall_wait", "stall_math", "stall_mio",
           "stall_not_selected", "stall_selected", "stall_lg", "stall_branch_resolving", "stall_dispatch",
           "stall_no_inst", "stall_tex", "stall_drain", "stall_misc"]


def main(path, top=25):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    data = [r for r in rows[2:] if len(r) == len(h)]
    f = lambda r, k: float(r[ix[k]] or 0)  # noqa: E731
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
    print(f"samples {tot:.0f}")
    reason = collections.Counter()
    for r in data:
        for k in REASONS:
            if k in ix:
                reason[k] += f(r, k)
    print("by reason: " + ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in reason.most_common(10)))
    byop = collections.Counter()
    for r in data:
        op = re.sub(r"^@!?U?P\w+\s+", "", r[ix["Source"]].strip()).split(" ")[0]
        byop[op] += f(r, "Warp Stall Sampling (All Samples)")
    print("by opcode: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in byop.most_common(16)))
    print("top lines:")
    for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
        rs = sorted(((f(r, k), k[6:]) for k in REASONS if k in ix), reverse=True)[:2]
        print(f"  {r[ix['Address']][-5:]} {100 * f(r, 'Warp Stall Sampling (All Samples)') / tot:4.1f}%  "
              f"{r[ix['Source']].strip()[:60]:60s} {rs[0][1]}/{rs[1][1]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
