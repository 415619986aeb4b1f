"""Host-side cost of the end-to-end path: per-packet Python + ctypes + staging copy."""
import cProfile
import os
import pstats
import sys
import time
from fractions import Fraction

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import EventArray, SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import ReconstructionEngine  # noqa: E402

geom = SensorGeometry(640, 480)
n, P = 10_000_000, 10_000
ev = workloads.make("texture", geom, n, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
xh, yh, ph = pin(ev.x.view(np.int16)).view(np.uint16), pin(ev.y.view(np.int16)).view(np.uint16), pin(ev.p)
pk = [EventArray(ev.t[a:a + P], xh[a:a + P], yh[a:a + P], ph[a:a + P]) for a in range(0, n, P)]
eng = ReconstructionEngine(geom, params)
for rep in range(3):
    eng.reset()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for b in pk:
        eng.process_array(b)
    t1 = time.perf_counter()
    fr = eng.render("robust")
    t2 = time.perf_counter()
    print(f"host loop {1e3 * (t1 - t0):.2f} ms, render+sync {1e3 * (t2 - t1):.2f} ms, total {1e3 * (t2 - t0):.2f} ms")
eng.reset()
pr = cProfile.Profile()
pr.enable()
for b in pk:
    eng.process_array(b)
eng.render("robust")
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
