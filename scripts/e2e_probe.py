"""Where does the host-API (e2e) time go?  Times the per-packet host loop alone."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction
import numpy as np, torch
from paper_2510_20071_b200 import workloads
from paper_2510_20071_b200.core import SensorGeometry, compute_params, EventArray
from paper_2510_20071_b200.pipeline import ReconstructionEngine
geom = SensorGeometry(640, 480)
ev = workloads.moving_texture(640, 480, 4_000_000)
params = compute_params(40.0, Fraction(1, 2), geom)
eng = ReconstructionEngine(geom, params, batch_capacity=1 << 20)
xh = torch.from_numpy(ev.x.view(np.int16)).pin_memory().numpy().view(np.uint16)
yh = torch.from_numpy(ev.y.view(np.int16)).pin_memory().numpy().view(np.uint16)
ph = torch.from_numpy(ev.p).pin_memory().numpy()
P = 10000
pk = [EventArray(ev.t[a:a+P], xh[a:a+P], yh[a:a+P], ph[a:a+P]) for a in range(0, len(ev), P)]
for rep in range(3):
    eng.reset(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for b in pk:
        eng.process_array(b)
    t1 = time.perf_counter()
    eng.flush(); torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host loop {1e3*(t1-t0):.2f} ms ({1e6*(t1-t0)/len(pk):.1f} us/packet), total {1e3*(t2-t0):.2f} ms")
import ctypes as C
lib = eng._lib
x0 = xh.ctypes.data
t0 = time.perf_counter()
for a in range(0, len(ev), P):
    lib.fibar_process(eng._h, x0 + 2*a, yh.ctypes.data + 2*a, ph.ctypes.data + a, P, 0)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"raw ctypes loop {1e6*(t1-t0)/len(pk):.1f} us/packet")
