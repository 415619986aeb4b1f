import os, sys
os.environ["FIBAR_DEBUG_WINDOW"] = "1"
sys.path.insert(0, ".")
import numpy as np, torch
from fractions import Fraction
from paper_2510_20071_b200 import workloads
from paper_2510_20071_b200.core import SensorGeometry, compute_params
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine
geom = SensorGeometry(640, 480)
ev = workloads.moving_texture(640, 480, 2_100_000)
params = compute_params(40.0, Fraction(1, 2), geom)
eng = ReconstructionEngine(geom, params, batch_capacity=1 << 20)
xd = torch.from_numpy(ev.x.view(np.int16)).cuda(); yd = torch.from_numpy(ev.y.view(np.int16)).cuda(); pd = torch.from_numpy(ev.p).cuda()
for a in range(0, len(ev), 1 << 20):
    s0 = eng.stats()
    eng.process_array(DeviceEventArray(xd[a:a + (1 << 20)], yd[a:a + (1 << 20)], pd[a:a + (1 << 20)]))
    eng.flush()
    s1 = eng.stats()
    print("batch", a, {k: s1[k] - s0[k] for k in ("debug_window_bad", "window_reruns", "fix_rounds", "warm_pops", "window_chunks")})
