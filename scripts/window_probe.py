"""Window-speculation statistics under batch size / graph settings (scratch probe).

    python scripts/window_probe.py --kind texture_noise_hot --w 1280 --h 720 --events 3000000 CAP:GRAPHS ...
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
ap.add_argument("--events", type=int, default=3_000_000)
ap.add_argument("--kind", default="texture_noise_hot")
ap.add_argument("--w", type=int, default=1280)
ap.add_argument("--h", type=int, default=720)
ap.add_argument("--render-every", type=int, default=0, help="render after every k packets of 100k")
ap.add_argument("settings", nargs="+")
a = ap.parse_args()
geom = SensorGeometry(a.w, a.h)
ev = workloads.make(a.kind, geom, a.events, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
xd = torch.from_numpy(ev.x.view(np.int16)).cuda()
yd = torch.from_numpy(ev.y.view(np.int16)).cuda()
pd = torch.from_numpy(ev.p).cuda()
for s in a.settings:
    cap, graphs = s.split(":")
    os.environ["FIBAR_GRAPHS"] = graphs
    eng = ReconstructionEngine(geom, params, batch_capacity=int(cap))
    st0 = eng.stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P = 100_000
    for i, s0 in enumerate(range(0, a.events, P)):
        eng.process_array(DeviceEventArray(xd[s0:s0 + P], yd[s0:s0 + P], pd[s0:s0 + P]))
        if a.render_every and (i + 1) % a.render_every == 0:
            eng.render_device()
    eng.flush()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = eng.stats()
    print(f"cap {cap} graphs {graphs}: {dt * 1e3:.1f} ms, batches {st['batches']}, chunks {st['window_chunks']}, "
          f"reruns {st['window_reruns']}, fix_rounds {st['fix_rounds']}, warm_pops {st['warm_pops']}", flush=True)
    eng.close()
