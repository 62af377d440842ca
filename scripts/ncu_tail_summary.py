"""Summarise one full ncu capture of the cluster tail (k_tailsm): duration, registers, stall
ratios per issue, issue activity, eligible warps, and the executed-instruction mix by SASS
opcode (from the source page).  usage: python scripts/ncu_tail_summary.py rep.ncu-rep out.txt"""
import collections
import csv
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, r = rows[0], rows[2]
lines = []
for key in sorted(h):
    if key in ("gpu__time_duration.sum", "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
               "smsp__warps_eligible.avg.per_cycle_active", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active") \
            or key.startswith("smsp__average_warps_issue_stalled") and key.endswith("per_issue_active.ratio"):
        lines.append(f"{key} = {r[h.index(key)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
srows = list(csv.reader(src.splitlines()))
mix = collections.Counter()
if srows:
    hi = [i for i, x in enumerate(srows) if "Source" in x and any("Instructions Executed" in c for c in x)]
    if hi:
        hh = srows[hi[0]]
        si = hh.index("Source")
        ei = [i for i, c in enumerate(hh) if c.strip() == "Instructions Executed"][0]
        for x in srows[hi[0] + 1:]:
            if len(x) <= max(si, ei):
                continue
            op = x[si].strip().split()
            if not op:
                continue
            o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
            try:
                mix[o.split(".")[0]] += float(x[ei].replace(",", ""))
            except ValueError:
                pass
tot = sum(mix.values())
if tot:
    lines.append(f"# executed warp instructions per launch: {int(tot)}; mix (share):")
    lines.append(", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in mix.most_common(18)))
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
