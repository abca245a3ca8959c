#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

usage: launch_summary.py RAW.csv OUT_PREFIX "command line"
Writes OUT_PREFIX.csv (id, kernel, grid, block, ns: one row per launch) and
OUT_PREFIX.md (per-kernel launches, total, share, mean).  ncu serialises
launches and runs them cold-cache: compare shares, not absolute times.
"""
import collections
import csv
import sys


def main():
    raw, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = []
    with open(raw) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(
            r["Metric Unit"], 1.0)
        rows.append((int(r["ID"]), r["Kernel Name"], r["Grid Size"], r["Block Size"], ns * scale))
    with open(out + ".csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "block", "ns"])
        for row in rows:
            w.writerow([row[0], row[1], row[2], row[3], f"{row[4]:.0f}"])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for _, k, _, _, ns in rows:
        short = k.split("(")[0] if not k.startswith("void ") else k[5:].split("(")[0]
        agg[short][0] += 1
        agg[short][1] += ns
    total = sum(v[1] for v in agg.values())
    with open(out + ".md", "w") as f:
        f.write(f"# launch list: `{cmd}` under `ncu --metrics gpu__time_duration.sum "
                f"--clock-control none`\n\n")
        f.write("Cold-cache, serialised per-launch device times (compare shares, not absolutes). "
                f"{len(rows)} launches; raw per-launch rows: `{out.split('/')[-1]}.csv`.\n\n")
        f.write("| kernel | launches | total ms | share | mean ms/launch |\n|---|---|---|---|---|\n")
        for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| `{k[:90]}` | {n} | {ns / 1e6:.3f} | {100 * ns / total:.2f}% | "
                    f"{ns / n / 1e6:.4f} |\n")


if __name__ == "__main__":
    main()
