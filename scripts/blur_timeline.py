"""Debug: per-item completion timeline of the blur dataflow for one 1M batch."""
import os, sys
os.environ["FIBAR_DEBUG_TIMES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction
import numpy as np, torch
from paper_2510_20071_b200 import workloads, _native
from paper_2510_20071_b200.core import SensorGeometry, compute_params
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine
geom = SensorGeometry(640, 480)
ev = workloads.moving_texture(640, 480, 2 << 20)
params = compute_params(40.0, Fraction(1, 2), geom)
eng = ReconstructionEngine(geom, params, batch_capacity=1 << 20)
xd = torch.from_numpy(ev.x.view(np.int16)).cuda(); yd = torch.from_numpy(ev.y.view(np.int16)).cuda(); pd = torch.from_numpy(ev.p).cuda()
B = 1 << 20
for a in (0, B):
    st0 = eng.stats()
    eng.process_array(DeviceEventArray(xd[a:a + B], yd[a:a + B], pd[a:a + B]))
    eng.flush()
st1 = eng.stats()
npop = st1["pops"] - st0["pops"]
done = np.zeros(npop, np.uint64); grab = np.zeros(npop, np.uint64)
_native.check(eng._lib.fibar_debug_times(eng._h, done.ctypes.data, grab.ctypes.data, npop), "dbg")
m = done > 0
d = done[m].astype(np.float64)
t0 = d.min()
d = (d - t0) / 1e3
idx = np.nonzero(m)[0]
print("items", npop, "blurred", m.sum(), "span us", d.max())
order = np.argsort(d)
for f in (0.01, 0.1, 0.25, 0.5, 0.75, 0.9, 0.99, 0.999, 1.0):
    k = min(len(d) - 1, int(f * len(d)))
    print(f"{f:6.3f} of items done by {d[order[k]]:10.1f} us")
# completion time vs item index
for f in (0.1, 0.5, 0.9, 1.0):
    k = int(f * (len(idx) - 1))
    print(f"item rank {f}: index {idx[k]} done at {d[k]:.1f} us")
late = idx[d > np.percentile(d, 99.9)]
print("latest items (index):", late[:20])

prep = np.zeros((npop, 20), np.uint32)
_native.check(eng._lib.fibar_debug_prep(eng._h, prep.ctypes.data, npop), "prep")
okm, pend = prep[:, 0], prep[:, 1]
flags = prep[:, 2:11]
done_f = done.astype(np.float64)
hops = []; ndeps = []
for p_ in np.nonzero(okm)[0][::50]:
    fs = [int(flags[p_, t]) & 0x7FFFFFFF for t in range(9) if (pend[p_] >> t) & 1]
    ndeps.append(len(fs))
    if fs and done[p_] > 0:
        last = max(done_f[f] for f in fs)
        hops.append((done_f[p_] - last) / 1e3)
hops = np.array(hops)
print("pending taps per item: mean", np.mean(ndeps), "frac items with deps", np.mean(np.array(ndeps) > 0))
print("hop latency (done - last dep done) us percentiles 10/50/90/99:", np.percentile(hops, [10, 50, 90, 99]))
