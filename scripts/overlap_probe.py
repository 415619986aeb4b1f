"""Wall-clock (CUDA events) of one filter-ON pass under env knob settings.

    python scripts/overlap_probe.py --events 10000000 "FIBAR_SERIAL=1" "FIBAR_BLUR_BLOCKS=2" ...
Each setting is a space-separated list of VAR=VALUE applied before engine creation.
"""
import argparse
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

ap = argparse.ArgumentParser()
ap.add_argument("--events", type=int, default=10_000_000)
ap.add_argument("--cap", type=int, default=1 << 20)
ap.add_argument("--packet", type=int, default=10_000)
ap.add_argument("--kind", default="texture")
ap.add_argument("--w", type=int, default=640)
ap.add_argument("--h", type=int, default=480)
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--noblur", action="store_true", help="blur_enabled=False (front-end cost alone)")
ap.add_argument("--profile", action="store_true", help="also print per-kernel ms from one profiled pass")
ap.add_argument("settings", nargs="+")
a = ap.parse_args()
geom = SensorGeometry(a.w, a.h)
ev = workloads.make(a.kind, geom, a.events, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
xd = torch.from_numpy(ev.x.view(np.int16)).cuda()
yd = torch.from_numpy(ev.y.view(np.int16)).cuda()
pd = torch.from_numpy(ev.p).cuda()
packets = [DeviceEventArray(xd[i:i + a.packet], yd[i:i + a.packet], pd[i:i + a.packet])
           for i in range(0, a.events, a.packet)]
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
ref = None
for s in a.settings:
    env = dict(kv.split("=", 1) for kv in s.split())
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    eng = ReconstructionEngine(geom, params, batch_capacity=a.cap, blur_enabled=not a.noblur)
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    times = []
    for rep in range(a.reps):
        eng.reset()
        flush.fill_(rep)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        for p in packets:
            eng.process_array(p)
        eng.render_device()
        host_ms = (time.perf_counter() - h0) * 1e3
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    l = eng.l
    same = ref is None or np.array_equal(l, ref)
    ref = l if ref is None else ref
    best = min(times[1:]) if len(times) > 1 else times[0]
    print(f"{s:>40}: {best:8.3f} ms  ({a.events / best / 1e3:7.1f} Mev/s)  all={['%.2f' % t for t in times]} host_enqueue={host_ms:.2f} ms same={same}",
          flush=True)
    if a.profile:
        eng.reset()
        eng.profile(True)
        for p in packets:
            eng.process_array(p)
        eng.render_device()
        prof = eng.profile_read()
        eng.profile(False)
        tot = sum(v[0] for v in prof.values())
        print("    kernels (sum %.2f ms): " % tot + " ".join(f"{k}={v[0]:.3f}" for k, v in
                                                          sorted(prof.items(), key=lambda kv: -kv[1][0])), flush=True)
    eng.close()
