"""Per-step device time of the config-2 device arm (separate 10k-event packets), with the
window statistics of slow steps."""
import os, sys, time
from fractions import Fraction
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine  # noqa: E402
n, P = 10_000_000, 10_000
geom = SensorGeometry(640, 480)
ev = workloads.make_cached("texture", geom, n, seed=0)
params = compute_params(40.0, Fraction(1, 2), geom)
dpk = [DeviceEventArray(torch.from_numpy(ev.x[a:a + P].view(np.int16)).cuda(), torch.from_numpy(ev.y[a:a + P].view(np.int16)).cuda(),
                        torch.from_numpy(ev.p[a:a + P].copy()).cuda()) for a in range(0, n, P)]
eng = ReconstructionEngine(geom, params)
frame = torch.empty((480, 640), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
times = []
prev = eng.stats()
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 60):
    flush.zero_()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.reset()
    for blk in dpk:
        eng.process_array(blk)
    eng.render_device("robust", out=frame)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    st = eng.stats()
    times.append(ms)
    if ms > 12:
        print(f"step {rep}: {ms:.2f} ms  window_reruns {st['window_reruns']} warm_pops {st['warm_pops']} coop {st['coop_iters']} fix_rounds {st['fix_rounds']}")
t = np.array(times)
print(f"{len(t)} steps: median {np.median(t):.2f} ms, max {t.max():.2f} ms, >12 ms: {(t > 12).sum()}")
