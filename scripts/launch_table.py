"""Per-kernel totals of an ncu gpu__time_duration.sum launch list (CSV).

    python scripts/launch_table.py gpurun_out/launches.csv [units_divisor]
prints kernel, launches, total us, mean us, share.  `units_divisor`: divide
totals by this (e.g. the number of batches) for per-batch times.
"""
import collections
import csv
import io
import sys


def table(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("fibar::", "")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r["Metric Unit"], 1.0)
        tot[name] += v * scale
        cnt[name] += 1
    return tot, cnt


if __name__ == "__main__":
    tot, cnt = table(sys.argv[1])
    div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    allsum = sum(tot.values())
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k:28s} {cnt[k]:6d} {v / div:10.1f} {v / cnt[k]:8.2f} {100 * v / allsum:5.1f}%")
    print(f"total {allsum / div:.1f} us (/{div:g}), {sum(cnt.values())} launches")
