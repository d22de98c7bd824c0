"""Aggregate an ncu launch list (gpu__time_duration.sum per launch) by kernel:
count, total, mean and share of the step. Markdown on stdout.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/<name>.md
"""
import csv
import sys
from collections import defaultdict


def main(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3}.get(r["Metric Unit"], 1e-3)
        agg[name][0] += 1
        agg[name][1] += float(r["Metric Value"].replace(",", "")) * scale
    total = sum(v[1] for v in agg.values())
    print(f"ncu launch list `{path}` (cold-cache, serialised; compare shares)\n")
    print(f"total {total:.1f} us over {sum(v[0] for v in agg.values())} launches\n")
    print("| kernel | launches | total (us) | mean (us) | share |")
    print("|---|---|---|---|---|")
    for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {name} | {c} | {t:.1f} | {t / c:.2f} | {100 * t / total:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
