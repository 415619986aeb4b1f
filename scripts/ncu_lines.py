"""Warp-stall samples per CUDA source line of an ncu report (needs -lineinfo).

    python scripts/ncu_lines.py REPORT.ncu-rep SOURCE.cu [top]
"""
import csv
import io
import subprocess
import sys

rep, srcf = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
src = open(srcf).read().splitlines()
hdr, out, cur = None, {}, None
for r in rows:
    if len(r) >= 2 and r[0] in ("File Name", "File Path"):
        cur = r[1]
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-" and cur and cur.endswith(srcf.split("/")[-1]):
        d = dict(zip(hdr, r))
        try:
            s = int(d["Warp Stall Sampling (All Samples)"])
        except ValueError:
            continue
        if s:
            out[int(d["Line No"])] = out.get(int(d["Line No"]), 0) + s
tot = sum(out.values()) or 1
for l, s in sorted(out.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{s:6d} {100 * s / tot:5.1f}% L{l}: {src[l - 1].strip()[:110]}")
