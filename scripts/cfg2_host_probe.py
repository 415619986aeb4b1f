"""Config 2 host arm: where a step's time goes (process loop vs final render)."""
import os, sys, time
from fractions import Fraction
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import EventArray, SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import ReconstructionEngine  # noqa: E402
n = 10_000_000
geom = SensorGeometry(640, 480)
ev = workloads.make_cached("texture", geom, n, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
P = 10_000
xh = torch.from_numpy(ev.x.view(np.int16)).pin_memory().numpy().view(np.uint16)
yh = torch.from_numpy(ev.y.view(np.int16)).pin_memory().numpy().view(np.uint16)
ph = torch.from_numpy(ev.p).pin_memory().numpy()
pk = [EventArray(ev.t[a:a + P], xh[a:a + P], yh[a:a + P], ph[a:a + P]) for a in range(0, n, P)]
eng = ReconstructionEngine(geom, params)
for rep in range(4):
    eng.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    slow = []
    for i, blk in enumerate(pk):
        a = time.perf_counter()
        eng.process_array(blk)
        d = time.perf_counter() - a
        if d > 1e-3:
            slow.append((i, round(d * 1e3, 2)))
    t1 = time.perf_counter()
    f = eng.render("robust")
    t2 = time.perf_counter()
    print(f"rep {rep}: process loop {1e3 * (t1 - t0):.2f} ms, render {1e3 * (t2 - t1):.2f} ms, slow calls {slow[:12]}")
# the same after a device-arm pass on the same engine (bench order)
from paper_2510_20071_b200.pipeline import DeviceEventArray  # noqa: E402
dpk = [DeviceEventArray(torch.from_numpy(ev.x[a:a + P].view(np.int16)).cuda(), torch.from_numpy(ev.y[a:a + P].view(np.int16)).cuda(),
                        torch.from_numpy(ev.p[a:a + P].copy()).cuda()) for a in range(0, n, P)]
frame = torch.empty((480, 640), dtype=torch.uint8, device="cuda")
for rep in range(2):
    eng.reset()
    for blk in dpk:
        eng.process_array(blk)
    eng.render_device("robust", out=frame)
torch.cuda.synchronize()
for rep in range(3):
    eng.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, blk in enumerate(pk):
        eng.process_array(blk)
    t1 = time.perf_counter()
    f = eng.render("robust")
    t2 = time.perf_counter()
    print(f"after device arm, rep {rep}: process loop {1e3 * (t1 - t0):.2f} ms, render {1e3 * (t2 - t1):.2f} ms")
if os.environ.get("FIBAR_TRACE"):
    import ctypes as C
    cap = 100000
    b = np.zeros(cap, np.int64); lab = np.zeros(cap, np.int32); ms = np.zeros(cap, np.float64); nout = C.c_int64(0)
    eng._lib.fibar_debug_trace(eng._h, cap, b.ctypes.data, lab.ctypes.data, ms.ctypes.data, C.byref(nout))
    rows = {}
    for i in range(nout.value):
        rows.setdefault(int(b[i]), {})[int(lab[i])] = ms[i]
    ks = sorted(rows)
    for k in ks[:12] + ks[-24:]:
        r = rows[k]
        print(k, {l: round(v - rows[ks[0]].get(0, 0), 3) for l, v in sorted(r.items())})
