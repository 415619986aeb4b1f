"""Host time of the engine calls of the end-to-end arm (host packets, frames to pinned host memory)."""
import os, sys, time
from fractions import Fraction
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import EventArray, SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import ReconstructionEngine  # noqa: E402
n = 10_000_000
geom = SensorGeometry(1280, 720)
ev = workloads.make_cached("texture_noise_hot", geom, n, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
P = 100_000
xh = torch.from_numpy(ev.x.view(np.int16)).pin_memory().numpy().view(np.uint16)
yh = torch.from_numpy(ev.y.view(np.int16)).pin_memory().numpy().view(np.uint16)
ph = torch.from_numpy(ev.p).pin_memory().numpy()
pk = [EventArray(ev.t[a:a + P], xh[a:a + P], yh[a:a + P], ph[a:a + P]) for a in range(0, n, P)]
eng = ReconstructionEngine(geom, params)
outs = [torch.empty((720, 1280), dtype=torch.uint8, pin_memory=True) for _ in range(8)]
metas = [torch.empty(4, dtype=torch.float64, pin_memory=True) for _ in range(8)]
for rep in range(3):
    eng.reset()
    torch.cuda.synchronize()
    tp = tr = 0.0
    t0 = time.perf_counter()
    afs = []
    for i, blk in enumerate(pk):
        a = time.perf_counter()
        eng.process_array(blk)
        b = time.perf_counter()
        af = eng.render_async("robust", out=outs[i % 8], meta=metas[i % 8])
        c = time.perf_counter()
        tp += b - a
        tr += c - b
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: process_array {1e6 * tp / len(pk):.1f} us, render_async {1e6 * tr / len(pk):.1f} us, loop {1e6 * (t1 - t0) / len(pk):.1f}, wall {1e6 * (t2 - t0) / len(pk):.1f} us per packet")
