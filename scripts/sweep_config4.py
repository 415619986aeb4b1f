"""BASELINE config 4: packet-size sweep with a read-out after every packet.

1280x720 moving texture, filter ON and OFF, packets of 1k / 10k / 100k / 1M
events, robust read-out (render_device, frame stays in HBM) after each packet.
Reports Mev/s and the per-packet latency (process + read-out, CUDA events on
the stream) p50 / p99, plus the reference CPU path (C oracle port, one core)
on a short prefix of the same stream at the same cadence.

    python scripts/sweep_config4.py [--events 20000000] [--out profiles/TAG_config4_sweep.json]

The config's 50 M events are cut to a prefix per packet size (at most
--events and at most --max-packets packets) so the sweep fits a few minutes;
the JSON says what was run.
"""
import argparse
import json
import os
import sys
import time
from fractions import Fraction

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import SensorGeometry, compute_params  # noqa: E402
from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--events", type=int, default=20_000_000)
ap.add_argument("--max-packets", type=int, default=3000)
ap.add_argument("--cpu-seconds", type=float, default=4.0, help="CPU reference budget per point")
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "config4_sweep.json"))
ap.add_argument("--sync", action="store_true", help="render_device (read-out on the caller's stream) instead of "
                                                   "render_async (behind the blur stage, next packet overlapping)")
a = ap.parse_args()

geom = SensorGeometry(1280, 720)
ev = workloads.make("texture", geom, a.events, seed=0)
xd = torch.from_numpy(ev.x.view(np.int16)).cuda()
yd = torch.from_numpy(ev.y.view(np.int16)).cuda()
pd = torch.from_numpy(ev.p).cuda()
frame = torch.empty((geom.height, geom.width), dtype=torch.uint8, device="cuda")
meta = torch.empty(4, dtype=torch.float64, device="cuda")
rows = []
for spatial in (True, False):
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=spatial)
    for packet in (1_000, 10_000, 100_000, 1_000_000):
        n_pk = min(a.max_packets, a.events // packet)
        eng = ReconstructionEngine(geom, params)
        pk = [DeviceEventArray(xd[i * packet:(i + 1) * packet], yd[i * packet:(i + 1) * packet],
                               pd[i * packet:(i + 1) * packet]) for i in range(n_pk)]
        # warm-up pass, then the timed pass from a reset engine
        for p in pk[: min(20, n_pk)]:
            eng.process_array(p)
            eng.render_device("robust", out=frame)
        eng.reset()
        torch.cuda.synchronize()
        if a.sync:
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(n_pk + 1)]
            evs[0].record()
            for i, p in enumerate(pk):
                eng.process_array(p)
                eng.render_device("robust", out=frame)
                evs[i + 1].record()
            torch.cuda.synchronize()
            total_ms = evs[0].elapsed_time(evs[-1])
            lat = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(n_pk)]) * 1e3   # us per packet
        else:
            # packet i: from its submission on the stream to its frame in HBM
            starts = [torch.cuda.Event(enable_timing=True) for _ in range(n_pk)]
            ready = []
            for i, p in enumerate(pk):
                starts[i].record()
                eng.process_array(p)
                ready.append(eng.render_async("robust", out=frame, meta=meta).event)
            torch.cuda.synchronize()
            total_ms = starts[0].elapsed_time(ready[-1])
            lat = np.array([starts[i].elapsed_time(ready[i]) for i in range(n_pk)]) * 1e3
        # reference CPU path at the same cadence on a prefix
        from oracle import oracle as orc
        ref = orc.OracleEngine(geom.width, geom.height, params)
        t0 = time.perf_counter()
        done = 0
        while done < n_pk and time.perf_counter() - t0 < a.cpu_seconds:
            s, e = done * packet, (done + 1) * packet
            ref.process_array(ev.t[s:e], ev.x[s:e], ev.y[s:e], ev.p[s:e])
            ref.render("robust")
            done += 1
        cpu_s = time.perf_counter() - t0
        row = {"filter": "on" if spatial else "off", "packet": packet, "packets": n_pk, "events": n_pk * packet,
               "mev_s": n_pk * packet / total_ms / 1e3, "latency_us_p50": float(np.percentile(lat, 50)),
               "latency_us_p99": float(np.percentile(lat, 99)),
               "cpu_reference_mev_s": done * packet / cpu_s / 1e6 if done else None, "cpu_packets": done}
        rows.append(row)
        print(json.dumps(row), flush=True)
        eng.close()
out = {"config": "config4:1280x720 texture, robust read-out after every packet (%s)" %
       ("render_device, on the caller's stream" if a.sync else "render_async, behind the packet's blur stage"),
       "note": "prefix of the 50M-event stream per point (events/packets columns); latency = process + read-out "
               "per packet, CUDA events on the stream; CPU reference = C oracle port, one core, same cadence, "
               "time-boxed prefix", "rows": rows}
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump(out, open(a.out, "w"), indent=1)
print("wrote", a.out)
