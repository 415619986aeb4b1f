"""Debug: the blur dependency DAG of one 1M-event batch (config-2 texture):
pending taps per item, DAG depth, per-level time, and the hop latency from a
producer's completion to its consumer's (FIBAR_DEBUG_TIMES timestamps).

    python scripts/blur_dag.py           (set DAG_W, DAG_H, DAG_B, DAG_KIND to change the workload)
"""
import os
import sys

os.environ["FIBAR_DEBUG_TIMES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_20071_b200 import _native, workloads  # noqa: E402
from paper_2510_20071_b200.core import SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine  # noqa: E402

W, H = int(os.environ.get("DAG_W", 640)), int(os.environ.get("DAG_H", 480))
B = int(os.environ.get("DAG_B", 1 << 20))
geom = SensorGeometry(W, H)
ev = workloads.make(os.environ.get("DAG_KIND", "texture"), geom, 3 * B, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
eng = ReconstructionEngine(geom, params, batch_capacity=B)
xd = torch.from_numpy(ev.x.view(np.int16)).cuda()
yd = torch.from_numpy(ev.y.view(np.int16)).cuda()
pd = torch.from_numpy(ev.p).cuda()
for a in (0, B, 2 * B):
    st0 = eng.stats()
    eng.process_array(DeviceEventArray(xd[a:a + B], yd[a:a + B], pd[a:a + B]))
    eng.flush()
st1 = eng.stats()
npop = st1["pops"] - st0["pops"]
prep = np.zeros((npop, 12), np.uint32)
_native.check(eng._lib.fibar_debug_prep(eng._h, prep.ctypes.data, npop), "prep")
done = np.zeros(npop, np.uint64)
grab = np.zeros(npop, np.uint64)
_native.check(eng._lib.fibar_debug_times(eng._h, done.ctypes.data, grab.ctypes.data, npop), "times")
okm, pend, val = prep[:, 0], prep[:, 1], prep[:, 2:11]
items = np.nonzero(okm)[0]
print(f"pops {npop}, stale items {items.size}")
level = np.zeros(npop, np.int64)
n_item, n_run = 0, 0
for p in items:
    lv = 0
    for t in range(9):
        if (pend[p] >> t) & 1:
            w = int(val[p, t])
            if w & 0x80000000:
                n_run += 1          # a rebuilt-run position: its producer is not in the record
            else:
                n_item += 1
                lv = max(lv, level[w] + 1)
    level[p] = lv
print(f"pending taps: on blur items {n_item}, on rebuilt runs {n_run}; item-edge DAG depth {level.max() + 1}")
d = done.astype(np.float64)
g = grab.astype(np.float64)
ok = d > 0
t0 = d[ok].min()
print(f"blur span {(d[ok].max() - t0) / 1e3:.1f} us; us per item-edge level {(d[ok].max() - t0) / 1e3 / (level.max() + 1):.2f}")
hop, waited = [], 0
for p in items[::7]:
    last = 0.0
    for t in range(9):
        if (pend[p] >> t) & 1:
            w = int(val[p, t])
            if not w & 0x80000000:
                last = max(last, d[w])
    if last > 0 and d[p] > 0:
        if g[p] <= last:
            hop.append((d[p] - last) / 1e3)
        else:
            waited += 1
print("hop latency, consumer already taken when its last item producer finished (us) p10/50/90/99:",
      np.round(np.percentile(hop, [10, 50, 90, 99]), 2), f"(n={len(hop)}; taken later: {waited})")
