"""Host submission time vs device time of the bench's device arm (config 3 prefix).
usage: python scripts/host_rate.py [events]"""
import os
import sys
import time
from fractions import Fraction

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
mode = sys.argv[2] if len(sys.argv) > 2 else "render"   # render: a read-out per packet; flush: a batch per packet, no read-out
geom = SensorGeometry(1280, 720)
ev = workloads.make_cached("texture_noise_hot", geom, n, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
P = 100_000
pk = [DeviceEventArray(torch.from_numpy(ev.x[a:a + P].view(np.int16)).cuda(), torch.from_numpy(ev.y[a:a + P].view(np.int16)).cuda(),
                       torch.from_numpy(ev.p[a:a + P].copy()).cuda()) for a in range(0, n, P)]
eng = ReconstructionEngine(geom, params)
frame = torch.empty((720, 1280), dtype=torch.uint8, device="cuda")
meta = torch.empty(4, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
for rep in range(3):
    eng.reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    host = {"proc": 0.0, "render": 0.0}
    for blk in pk:
        a = time.perf_counter()
        eng.process_array(blk)
        b = time.perf_counter()
        if mode == "render":
            af = eng.render_async("robust", out=frame, meta=meta)
        else:
            eng.flush()
        host["proc"] += b - a
        host["render"] += time.perf_counter() - b
    t1 = time.perf_counter()
    if mode == "render":
        s.wait_event(af.event)
    else:
        eng.brightness_device()
    e1.record(s)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    nb = len(pk)
    print(f"rep {rep}: host loop {1e6 * (t1 - t0) / nb:.1f} us/batch (process_array {1e6 * host['proc'] / nb:.1f}, "
          f"render_async {1e6 * host['render'] / nb:.1f}), device {1e3 * e0.elapsed_time(e1) / nb:.1f} us/batch, "
          f"wall {1e6 * (t2 - t0) / nb:.1f} us/batch")
