"""Per-batch stream-part marks of a large-batch config (FIBAR_TRACE): config 2 device arm."""
import ctypes as C, os, sys
from fractions import Fraction
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FIBAR_TRACE"] = "1"
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine  # noqa: E402
w, h, n, kind = (640, 480, 10_000_000, "texture") if len(sys.argv) < 2 else (2560, 1440, 30_000_000, "texture")
geom = SensorGeometry(w, h)
ev = workloads.make_cached(kind, geom, n, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
xd = torch.from_numpy(ev.x.view(np.int16)).cuda(); yd = torch.from_numpy(ev.y.view(np.int16)).cuda(); pd = torch.from_numpy(ev.p).cuda()
eng = ReconstructionEngine(geom, params)
frame = torch.empty((h, w), dtype=torch.uint8, device="cuda")
for rep in range(3):
    eng.reset()
    eng.process_array(DeviceEventArray(xd, yd, pd))
    eng.render_device("robust", out=frame)
    torch.cuda.synchronize()
cap = 100000
b = np.zeros(cap, np.int64); lab = np.zeros(cap, np.int32); ms = np.zeros(cap, np.float64); nout = C.c_int64(0)
eng._lib.fibar_debug_trace(eng._h, cap, b.ctypes.data, lab.ctypes.data, ms.ctypes.data, C.byref(nout))
rows = {}
for i in range(nout.value):
    rows.setdefault(int(b[i]), {})[int(lab[i])] = ms[i]
ks = sorted(rows)[-10:]
t0 = rows[ks[0]][0]
print("batch  ingest_beg ingest_end  blur_beg  blur_end   (ms)")
for k in ks:
    r = rows[k]
    print(k, " ".join(f"{r.get(l, float('nan')) - t0:9.3f}" for l in (0, 1, 6, 7)))
