"""Per-kernel time of one small packet + read-out (config-4 style), filter ON and OFF."""
import os
import sys
from fractions import Fraction

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
geom = SensorGeometry(1280, 720)
ev = workloads.make("texture", geom, 200 * P, seed=0)
xd = torch.from_numpy(ev.x.view(np.int16)).cuda()
yd = torch.from_numpy(ev.y.view(np.int16)).cuda()
pd = torch.from_numpy(ev.p).cuda()
frame = torch.empty((720, 1280), dtype=torch.uint8, device="cuda")
for spatial in (True, False):
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=spatial)
    eng = ReconstructionEngine(geom, params)
    for i in range(100):
        eng.process_array(DeviceEventArray(xd[i * P:(i + 1) * P], yd[i * P:(i + 1) * P], pd[i * P:(i + 1) * P]))
        eng.render_device("robust", out=frame)
    torch.cuda.synchronize()
    eng.profile(True)
    for i in range(100, 200):
        eng.process_array(DeviceEventArray(xd[i * P:(i + 1) * P], yd[i * P:(i + 1) * P], pd[i * P:(i + 1) * P]))
        eng.render_device("robust", out=frame)
    prof = eng.profile_read()
    eng.profile(False)
    tot = sum(v[0] for v in prof.values()) / 100
    print(f"filter {'ON' if spatial else 'OFF'} packet {P}: kernel-sum {tot * 1e3:.1f} us per packet:",
          " ".join(f"{k}={v[0] / 100 * 1e3:.1f}" for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])))
    eng.close()
