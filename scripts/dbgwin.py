"""FIBAR_DEBUG_WINDOW: recount every chunk's anchor counts serially and report
mismatches per batch (plus verifier re-runs / rounds).

    python scripts/dbgwin.py [kind W H events cap]
"""
import os
import sys
os.environ["FIBAR_DEBUG_WINDOW"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from fractions import Fraction  # noqa: E402
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "texture"
W, H = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (640, 480)
n = int(sys.argv[4]) if len(sys.argv) > 4 else 2_100_000
cap = int(sys.argv[5]) if len(sys.argv) > 5 else 1 << 20
geom = SensorGeometry(W, H)
ev = workloads.make(kind, geom, n, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
eng = ReconstructionEngine(geom, params, batch_capacity=cap)
xd = torch.from_numpy(ev.x.view(np.int16)).cuda()
yd = torch.from_numpy(ev.y.view(np.int16)).cuda()
pd = torch.from_numpy(ev.p).cuda()
for a in range(0, len(ev), cap):
    s0 = eng.stats()
    q0 = eng.qs
    eng.process_array(DeviceEventArray(xd[a:a + cap], yd[a:a + cap], pd[a:a + cap]))
    eng.flush()
    s1 = eng.stats()
    print("batch", a, "qlen/target", int(q0[1]), int(q0[2]),
          {k: s1[k] - s0[k] for k in ("debug_window_bad", "window_reruns", "fix_rounds", "warm_pops", "window_chunks")},
          flush=True)
