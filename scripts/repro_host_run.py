"""Host packets through run() with a read-out per packet (the bench's e2e arm),
checked frame by frame against the oracle.  usage: python scripts/repro_host_run.py [events] [packet] [steps]"""
import os
import sys
from fractions import Fraction

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import EventArray, SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import ReconstructionEngine, run  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
P = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
geom = SensorGeometry(1280, 720)
ev = workloads.make_cached("texture_noise_hot", geom, n, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
cuts = list(range(0, n, P)) + [n]
xh = torch.from_numpy(ev.x.view(np.int16)).pin_memory().numpy().view(np.uint16)
yh = torch.from_numpy(ev.y.view(np.int16)).pin_memory().numpy().view(np.uint16)
ph = torch.from_numpy(ev.p).pin_memory().numpy()
pk = [EventArray(ev.t[a:b], xh[a:b], yh[a:b], ph[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
times = [int(ev.t[b - 1]) + 1 for b in cuts[1:]]
# run() semantics: the frame at r holds exactly the events with t < r
ref = orc.OracleEngine(1280, 720, params)
want = []
done = 0
for r in times:
    upto = int(np.searchsorted(ev.t, np.uint64(r), side="left"))
    if upto > done:
        ref.process_array(ev.t[done:upto], ev.x[done:upto], ev.y[done:upto], ev.p[done:upto])
        done = upto
    want.append(ref.render("robust")[0])
eng = ReconstructionEngine(geom, params)
for s in range(steps):
    eng.reset()
    got = []
    run(eng, pk, readout_times=times, frame_sink=lambda k, f: got.append(f.pixels.copy()))
    bad = [k for k, (a, b) in enumerate(zip(got, want)) if not np.array_equal(a, b)]
    print(f"step {s}: {len(got)} frames, mismatches {bad[:8]}")
print("ok")
