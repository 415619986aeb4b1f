"""cProfile of the end-to-end arm (pipeline.run() over pinned host packets, a frame per packet)
usage: python scripts/e2e_profile.py [events]"""
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
from paper_2510_20071_b200.pipeline import ReconstructionEngine, run  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
geom = SensorGeometry(1280, 720)
ev = workloads.make_cached("texture_noise_hot", geom, n, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
P = 100_000
cuts = list(range(0, n, P)) + [n]
xh = torch.from_numpy(ev.x.view(np.int16)).pin_memory().numpy().view(np.uint16)
yh = torch.from_numpy(ev.y.view(np.int16)).pin_memory().numpy().view(np.uint16)
ph = torch.from_numpy(ev.p).pin_memory().numpy()
pk = [EventArray(ev.t[a:b], xh[a:b], yh[a:b], ph[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
times = [int(ev.t[b - 1]) + 1 for b in cuts[1:]]
eng = ReconstructionEngine(geom, params)
last = {}


def step():
    eng.reset()
    run(eng, pk, readout_times=times, frame_sink=lambda k, f: last.__setitem__("f", f))
    torch.cuda.synchronize()


step()
for _ in range(2):
    t0 = time.perf_counter()
    step()
    dt = time.perf_counter() - t0
    print(f"run(): {1e6 * dt / len(pk):.1f} us per packet, {n / dt / 1e6:.1f} Mev/s")
pr = cProfile.Profile()
pr.enable()
step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
