"""Summarise ncu outputs (launch list CSV + full-capture report) into profiles/."""
import collections
import csv
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        key = (r[ki].split("(")[0].strip(), r[gi])
        a = agg.setdefault(key, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)",
           f"# total device time {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches",
           f"{'kernel':70s} {'grid':>16s} {'n':>6s} {'total_ms':>10s} {'avg_us':>10s} {'share':>6s}"]
    for (k, g), (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k[:70]:70s} {g:>16s} {n:6d} {t / 1e6:10.3f} {t / n / 1e3:10.2f} {t / tot:6.3f}")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
            "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
    out = ["# ncu --set full --clock-control none (one capture per listed launch)",
           "# units: " + ", ".join(f"{w}={u[h.index(w)]}" for w in want if w in h)]
    recs = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        stalls = []
        for k, v in d.items():
            if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        s = sum(v for v, _ in stalls) or 1
        rec = {"kernel": d["Kernel Name"].split("(")[0], "grid": d["Grid Size"], "block": d["Block Size"]}
        for w in want:
            rec[w] = d.get(w)
        rec["top_stalls"] = ", ".join(f"{k}={v / s:.2f}" for v, k in stalls[:4])
        recs.append(rec)
        out.append(json.dumps(rec))
    return "\n".join(out), recs


if __name__ == "__main__":
    # usage: summarize_ncu.py TAG LAUNCH_CSV|- REPORT.ncu-rep
    tag, lcsv, rep = sys.argv[1], sys.argv[2], sys.argv[3]
    if lcsv != "-":
        open(f"profiles/{tag}_launches.txt", "w").write(launches(lcsv) + "\n")
        print(open(f"profiles/{tag}_launches.txt").read()[:3000])
    txt, recs = full(rep)
    open(f"profiles/{tag}_ncu_full.txt", "w").write(txt + "\n")
    print(txt[:6000])
