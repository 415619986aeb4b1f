"""Host-path variants of a per-packet read-out loop (config 3 shape), wall clock:
process+render (sync), process+render_async, run() (pipelined frames)."""
import os
import sys
import time
from fractions import Fraction

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import EventArray, SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import ReconstructionEngine, run  # noqa: E402

geom = SensorGeometry(1280, 720)
ev = workloads.make("texture_noise_hot", geom, 3_000_000, seed=0)
eng = ReconstructionEngine(geom, compute_params(40.0, Fraction(1, 2), geom))
P = 100_000
xh = torch.from_numpy(ev.x.view(np.int16)).pin_memory().numpy().view(np.uint16)
yh = torch.from_numpy(ev.y.view(np.int16)).pin_memory().numpy().view(np.uint16)
ph = torch.from_numpy(ev.p).pin_memory().numpy()
cuts = list(range(0, len(ev), P)) + [len(ev)]
pk = [EventArray(ev.t[a:b], xh[a:b], yh[a:b], ph[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
times = [int(ev.t[b - 1]) + 1 for b in cuts[1:]]
last = {}


def v_sync():
    eng.reset()
    for b in pk:
        eng.process_array(b)
        last["f"] = eng.render("robust")


def v_async():
    eng.reset()
    q = []
    for b in pk:
        eng.process_array(b)
        q.append(eng.render_async("robust"))
        if len(q) > 4:
            last["f"] = q.pop(0).frame()
    for a in q:
        last["f"] = a.frame()


def v_run():
    eng.reset()
    run(eng, pk, readout_times=times, frame_sink=lambda k, f: last.__setitem__("f", f))


for name, fn in (("sync", v_sync), ("async", v_async), ("run", v_run)):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms per 3M events ({len(pk)} packets)", flush=True)
if len(sys.argv) > 1:
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    v_run()
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)

# host time of the native calls alone (no GPU waits: the engine is far ahead)
tp, tr = 0.0, 0.0
eng.reset()
torch.cuda.synchronize()
for b in pk:
    t0 = time.perf_counter()
    eng.process_array(b)
    t1 = time.perf_counter()
    eng.render_async("robust")
    tr += time.perf_counter() - t1
    tp += t1 - t0
torch.cuda.synchronize()
print(f"host per packet: process_array {tp / len(pk) * 1e6:.0f} us, render_async {tr / len(pk) * 1e6:.0f} us")
