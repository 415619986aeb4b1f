"""Per-batch timeline of the streamed schedule (FIBAR_TRACE=1): durations of
each stream part and the waits between them, averaged over steady-state
batches of a config-3 prefix with a read-out per packet.
usage: FIBAR_TRACE=1 python scripts/trace_parts.py [events]"""
import collections
import ctypes as C
import os
import sys
from fractions import Fraction

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FIBAR_TRACE"] = "1"
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6_000_000
geom = SensorGeometry(1280, 720)
ev = workloads.make_cached("texture_noise_hot", geom, n, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
P = 100_000
pk = [DeviceEventArray(torch.from_numpy(ev.x[a:a + P].view(np.int16)).cuda(), torch.from_numpy(ev.y[a:a + P].view(np.int16)).cuda(),
                       torch.from_numpy(ev.p[a:a + P].copy()).cuda()) for a in range(0, n, P)]
eng = ReconstructionEngine(geom, params)
frame = torch.empty((720, 1280), dtype=torch.uint8, device="cuda")
meta = torch.empty(4, dtype=torch.float64, device="cuda")
for rep in range(2):
    eng.reset()
    for blk in pk:
        eng.process_array(blk)
        eng.render_async("robust", out=frame, meta=meta)
    torch.cuda.synchronize()
    cap = 100000
    b = np.zeros(cap, np.int64)
    lab = np.zeros(cap, np.int32)
    ms = np.zeros(cap, np.float64)
    nout = C.c_int64(0)
    eng._lib.fibar_debug_trace(eng._h, cap, b.ctypes.data, lab.ctypes.data, ms.ctypes.data, C.byref(nout))
n_ = nout.value
t = collections.defaultdict(dict)
b0 = b[0]
for i in range(n_):
    t[int(b[i] - b0)][int(lab[i])] = ms[i] * 1e3   # us
ks = sorted(k for k in t if 10 <= k < max(t) - 2 and all(l in t[k] for l in range(9)))
def avg(f):
    v = [f(k) for k in ks if (k + 1) in t]
    return float(np.mean(v)) if v else float("nan")
print(f"{len(ks)} steady batches (us per batch, means)")
print(f"period (window start k -> k+1): {avg(lambda k: t[k + 1][2] - t[k][2]):.1f}")
print(f"ingest       {avg(lambda k: t[k][1] - t[k][0]):.1f}   starts {avg(lambda k: t[k][0] - t[k][2]):+.1f} vs its window start")
print(f"window part  {avg(lambda k: t[k][3] - t[k][2]):.1f}   waits {avg(lambda k: t[k + 1][2] - t[k][3]):.1f} before the next")
print(f"  window start - ingest end   {avg(lambda k: t[k][2] - t[k][1]):.1f}")
print(f"eviction     {avg(lambda k: t[k][5] - t[k][4]):.1f}   starts {avg(lambda k: t[k][4] - t[k][3]):+.1f} after the window part")
print(f"blur stage   {avg(lambda k: t[k][7] - t[k][6]):.1f}   starts {avg(lambda k: t[k][6] - t[k][5]):+.1f} after the eviction pass; "
      f"{avg(lambda k: t[k][6] - t[k - 1][8]):+.1f} after the previous read-out")
print(f"read-out     {avg(lambda k: t[k][8] - t[k][7]):.1f}")
if os.environ.get("TRACE_ROWS"):
    # raw rows: every mark of a few consecutive steady batches, relative to the first one's ingest start
    k0 = ks[len(ks) // 2]
    base = t[k0][0]
    print("batch  " + "  ".join(f"{n:>9s}" for n in ("ing_beg", "ing_end", "win_beg", "win_end", "evi_beg", "evi_end", "blur_beg", "blur_end", "readout")))
    for k in range(k0, k0 + 8):
        if k in t:
            print(f"{k:5d}  " + "  ".join(f"{t[k].get(l, float('nan')) - base:9.1f}" for l in range(9)))
