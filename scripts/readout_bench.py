"""Device time of one read-out (render_device, robust and fixed) at 1280x720
and 2560x1440, CUDA events over 200 back-to-back frames."""
import os
import sys
from fractions import Fraction

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import ReconstructionEngine  # noqa: E402

for w, h in ((1280, 720), (2560, 1440), (640, 480)):
    geom = SensorGeometry(w, h)
    ev = workloads.make("texture", geom, 2_000_000, seed=0)
    eng = ReconstructionEngine(geom, compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=True))
    eng.process_array(ev)
    frame = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    for mode in ("robust", "fixed"):
        for _ in range(20):
            eng.render_device(mode, out=frame)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(200):
            eng.render_device(mode, out=frame)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 200 * 1e3
        print(f"{w}x{h} {mode}: {us:.1f} us per read-out ({w * h * 5 / us / 1e3:.0f} GB/s at 5 B/pixel)")
    eng.close()

# phase stamps of one 1280x720 robust read-out (needs a FIBAR_RO_TIMES build, FIBAR_LIB)
if os.environ.get("FIBAR_LIB"):
    import ctypes as C
    geom = SensorGeometry(1280, 720)
    ev = workloads.make("texture", geom, 2_000_000, seed=0)
    eng = ReconstructionEngine(geom, compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=True))
    eng.process_array(ev)
    frame = torch.empty((720, 1280), dtype=torch.uint8, device="cuda")
    for _ in range(5):
        eng.render_device("robust", out=frame)
        torch.cuda.synchronize()
        ts = (C.c_uint64 * 16)()
        eng._lib.fibar_debug_readout_times(eng._h, ts)
        t0 = ts[1]
        print("phase stamps (ns from CTA 0 start):", [int(ts[k] - t0) if ts[k] else None for k in range(1, 16)])

