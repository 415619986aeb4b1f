"""Which part of a device-arm pass makes later small-batch graph captures slow (config 2 host arm)."""
import os, sys, time
from fractions import Fraction
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import EventArray, SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine  # noqa: E402
mode = sys.argv[1]
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
frame = torch.empty((480, 640), dtype=torch.uint8, device="cuda")
if mode == "alloc":
    dpk = [torch.empty(10000, dtype=torch.int16, device="cuda") for _ in range(3000)]
elif mode in ("views", "separate"):
    if mode == "views":
        xd = torch.from_numpy(ev.x.view(np.int16)).cuda(); yd = torch.from_numpy(ev.y.view(np.int16)).cuda(); pd = torch.from_numpy(ev.p).cuda()
        dpk = [DeviceEventArray(xd[a:a + P], yd[a:a + P], pd[a:a + P]) for a in range(0, n, P)]
    else:
        dpk = [DeviceEventArray(torch.from_numpy(ev.x[a:a + P].view(np.int16)).cuda(), torch.from_numpy(ev.y[a:a + P].view(np.int16)).cuda(),
                                torch.from_numpy(ev.p[a:a + P].copy()).cuda()) for a in range(0, n, P)]
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
    for blk in pk:
        eng.process_array(blk)
    t1 = time.perf_counter()
    f = eng.render("robust")
    t2 = time.perf_counter()
    print(f"{mode} rep {rep}: process loop {1e3 * (t1 - t0):.2f} ms, render {1e3 * (t2 - t1):.2f} ms")
