"""N packets of P events (1280x720 texture) with a robust read-out after each, no profiling
hooks (CUDA graphs on): the command to put under an ncu launch list for config 4.

    python scripts/small_packets.py P N [on|off]
"""
import os
import sys
from fractions import Fraction

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine  # noqa: E402

P = int(sys.argv[1])
N = int(sys.argv[2])
spatial = (sys.argv[3] if len(sys.argv) > 3 else "on") == "on"
geom = SensorGeometry(1280, 720)
ev = workloads.make("texture", geom, 2 * N * P, seed=0)
xd = torch.from_numpy(ev.x.view(np.int16)).cuda()
yd = torch.from_numpy(ev.y.view(np.int16)).cuda()
pd = torch.from_numpy(ev.p).cuda()
frame = torch.empty((720, 1280), dtype=torch.uint8, device="cuda")
eng = ReconstructionEngine(geom, compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=spatial))
for i in range(2 * N):
    if i == N:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    eng.process_array(DeviceEventArray(xd[i * P:(i + 1) * P], yd[i * P:(i + 1) * P], pd[i * P:(i + 1) * P]))
    eng.render_device("robust", out=frame)
e1.record()
torch.cuda.synchronize()
print(f"packet {P} filter {'on' if spatial else 'off'}: {e0.elapsed_time(e1) / N * 1e3:.1f} us per packet incl. read-out")
