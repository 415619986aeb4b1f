"""Summarise ncu outputs into profiles/ (tracked).

    python scripts/summarize_ncu.py TAG "WORKLOAD CLASS" DEVICE_BATCH_CAP "COMMAND" [BATCHES]
reads gpurun_out/launches_TAG.csv (gpu__time_duration.sum launch list) and
gpurun_out/full_TAG.ncu-rep (--set full capture), writes profiles/TAG_launches.md,
profiles/TAG_ncu_full.md and profiles/TAG_traffic.json (per-launch DRAM bytes,
tagged with the workload class -- bench.py's workload string without the event
count -- and the device batch capacity, which bench.py matches before using it).
"""
import collections
import re
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
wclass = sys.argv[2] if len(sys.argv) > 2 else ""
bcap = int(sys.argv[3]) if len(sys.argv) > 3 else 0
command = sys.argv[4] if len(sys.argv) > 4 else ""
nbatches = float(sys.argv[5]) if len(sys.argv) > 5 else 0.0
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)

# launch list
path = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
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
    unit = r["Metric Unit"]
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    tot[name] += v * scale
    cnt[name] += 1
ours = {k: v for k, v in tot.items() if k.startswith("k_")}
allsum = sum(ours.values())
with open(os.path.join(out_dir, f"{tag}_launches.md"), "w") as fh:
    fh.write(f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
    fh.write(f"Command: `{command}`. Workload class: {wclass}; device batch capacity {bcap}. "
             "Per-launch times are cold-cache and serialised (ncu replays each kernel alone); "
             "compare shares, not absolutes.\n\n")
    fh.write("| kernel | launches | total us | mean us | share of our kernels |\n|---|---:|---:|---:|---:|\n")
    for k, v in sorted(ours.items(), key=lambda kv: -kv[1]):
        fh.write(f"| {k} | {cnt[k]} | {v:.1f} | {v / cnt[k]:.1f} | {v / allsum * 100:.1f}% |\n")
    fh.write(f"\nTotal of our kernels: {allsum:.1f} us over {sum(cnt[k] for k in ours)} launches"
             + (f" ({allsum / nbatches:.1f} us per device batch over {nbatches:g} batches)" if nbatches else "") + ".\n")
print("wrote launches summary;", len(ours), "kernels")

# full capture
rep = os.path.join(ROOT, "gpurun_out", f"full_{tag}.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
            "Compute (SM) Throughput", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
            "Executed Ipc Active", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
            "Grid Size", "Block Size"]
    per = collections.OrderedDict()
    for r in rows[1:]:
        k = (r[idx["ID"]], r[idx["Kernel Name"]].split("(")[0].replace("<unnamed>::", "").replace("fibar::", ""))
        if r[idx["Metric Name"]] in want:
            per.setdefault(k, {})[r[idx["Metric Name"]]] = f"{r[idx['Metric Value']]} {r[idx['Metric Unit']]}".strip()
    raw2 = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r2 = list(csv.reader(io.StringIO(raw2)))
    h2 = {h: i for i, h in enumerate(r2[0])}
    dram = {}
    for r in r2[2:]:
        try:
            k = r[h2["ID"]]
            rb = float(r[h2["dram__bytes_read.sum"]].replace(",", ""))
            wb = float(r[h2["dram__bytes_write.sum"]].replace(",", ""))
            unit_r = r2[1][h2["dram__bytes_read.sum"]]
            dram[k] = (rb, wb, unit_r)
        except (KeyError, ValueError, IndexError):
            pass
    with open(os.path.join(out_dir, f"{tag}_ncu_full.md"), "w") as fh:
        fh.write(f"# {tag}: ncu --set full (--clock-control none), top kernels of one bench step\n\n")
        fh.write("ncu flushes caches between replays, so DRAM traffic here is cold-cache (upper bound).\n\n")
        for (kid, name), m in per.items():
            fh.write(f"## {name} (launch id {kid})\n\n")
            for w in want:
                if w in m:
                    fh.write(f"- {w}: {m[w]}\n")
            if kid in dram:
                rb, wb, u = dram[kid]
                fh.write(f"- dram__bytes_read.sum + dram__bytes_write.sum: {rb:.3f} + {wb:.3f} {u}\n")
            fh.write("\n")
    # per-launch DRAM bytes by kernel (bench.py fills roofline.traffic from this)
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    traffic = {}
    for (kid, name), m in per.items():
        if kid in dram:
            rb, wb, u = dram[kid]
            short = re.sub(r"_g\d+$", "", name.replace("k_", "", 1))   # (k_window_run_g8 is launched as "window_run")
            traffic.setdefault(short, []).append((rb + wb) * scale.get(u, 1.0))
    import json
    with open(os.path.join(out_dir, f"{tag}_traffic.json"), "w") as fh:
        json.dump({"source": f"ncu --set full capture full_{tag}.ncu-rep (cold cache, one launch each)",
                   "workload_class": wclass, "device_batch_cap": bcap,
                   "bytes_per_launch": {k: sum(v) / len(v) for k, v in traffic.items()}}, fh, indent=1)
    print("wrote full summary;", len(per), "kernels")
