"""Sweep the window-speculation knobs (env vars read at engine creation) on one workload.

    python scripts/tune_window.py --events 4000000 --cap 1048576 CHUNK:WARM ...
Prints per setting: step ms, window kernel ms, warm pops/chunk, reruns, verifier rounds.
"""
import argparse
import os
import sys
from fractions import Fraction

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--events", type=int, default=4_000_000)
ap.add_argument("--cap", type=int, default=1 << 20)
ap.add_argument("--w", type=int, default=640)
ap.add_argument("--h", type=int, default=480)
ap.add_argument("--kind", default="texture")
ap.add_argument("settings", nargs="+")
a = ap.parse_args()
geom = SensorGeometry(a.w, a.h)
ev = workloads.make(a.kind, geom, a.events, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
xd = torch.from_numpy(ev.x.view(np.int16)).cuda()
yd = torch.from_numpy(ev.y.view(np.int16)).cuda()
pd = torch.from_numpy(ev.p).cuda()
ref_l = None
for s in a.settings:
    c, w = s.split(":")[:2]
    parts = s.split(":")
    dbg = parts[2] if len(parts) > 2 else "0"
    os.environ.update(FIBAR_CHUNK=c, FIBAR_WARM=w, FIBAR_DEBUG_WINDOW=dbg,
                      FIBAR_BLUR_BLOCKS=parts[3] if len(parts) > 3 else "64",
                      FIBAR_BLUR_SLEEP=parts[4] if len(parts) > 4 else "0",
                      FIBAR_BLUR_MODE=parts[5] if len(parts) > 5 else "1")
    eng = ReconstructionEngine(geom, params, batch_capacity=a.cap)
    for rep in range(2):
        eng.reset()
        st0 = eng.stats()
        eng.profile(True)
        eng.process_array(DeviceEventArray(xd, yd, pd))
        eng.flush()
        prof = eng.profile_read()
        eng.profile(False)
        st1 = eng.stats()
    tot = sum(v[0] for v in prof.values())
    win = sum(prof.get(k, (0, 0))[0] for k in ("anchor", "anchor_scan", "fp", "anchor2", "window_run", "window_fix"))
    ch = st1["window_chunks"] - st0["window_chunks"]
    l = eng.l
    same = ref_l is None or np.array_equal(l, ref_l)
    tb = prof.get('blur_prep', (0, 0))[0]
    ref_l = l if ref_l is None else ref_l
    detail = " ".join(f"{k}={prof[k][0]:.2f}" for k in ("anchor", "anchor_scan", "fp", "anchor2", "rs_scan", "rs_scatter", "blur_prep", "temporal", "link") if k in prof)
    print(detail)
    print(f"{s:>20}: step {tot:8.2f} ms  window {win:8.2f} ms (run {prof['window_run'][0]:.2f} fix {prof['window_fix'][0]:.2f})"
          f"  warm pops/chunk {(st1['warm_pops'] - st0['warm_pops']) / max(ch, 1):8.1f}  reruns {st1['window_reruns'] - st0['window_reruns']}"
          f"  rounds {st1['fix_rounds'] - st0['fix_rounds']}  blur {prof['blur'][0]:.2f} ms prep {tb:.2f}  same={same}", flush=True)
    eng.close()
