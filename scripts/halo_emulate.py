"""Filter-ON halo row bands emulated on one GPU: rounds and per-rank device time.

Measurement tool, not on the product path.  N native halo-band engines share
one GPU in one process (bands.run_local_halo_bands: rounds in lockstep, the
exchange as device copies; no kernel waits on another rank's, so this is safe
on one GPU).  Each rank's calls are bracketed with CUDA events, giving its
device-busy time per batch; ``projected_ms`` = sum over batches of the
slowest rank's busy time, i.e. an N-GPU step without exchange latency.  The
result is checked against a single-engine run of the same stream.

    python scripts/halo_emulate.py --config 2 --events 10000000 --bands 1,2,4,8 --halo 8 --batch 262144
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from fractions import Fraction

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2510_20071_b200 import bands, workloads
    from paper_2510_20071_b200.core import compute_params
    from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--events", type=int, default=None)
    ap.add_argument("--bands", default="1,2,4,8")
    ap.add_argument("--halo", default="8")
    ap.add_argument("--batch", default=str(1 << 18))
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = workloads.CONFIGS[a.config]
    geom = cfg["geometry"]
    n = a.events or cfg["n"]
    kw = {"speed": cfg["speed"]} if "speed" in cfg else {}
    ev = workloads.make(cfg["kind"], geom, n, seed=0, **kw)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=True)
    dev = torch.device("cuda", 0)
    xd = torch.from_numpy(ev.x.view(np.int16)).to(dev)
    yd = torch.from_numpy(ev.y.view(np.int16)).to(dev)
    pd = torch.from_numpy(ev.p).to(dev)
    # single-engine reference result and time (the normal overlapped path)
    ref = ReconstructionEngine(geom, params)
    for _ in range(2):
        ref.reset()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(0, n, 10_000):
            ref.process_array(DeviceEventArray(xd[s:s + 10_000], yd[s:s + 10_000], pd[s:s + 10_000]))
        ref.flush()
        e1.record()
        torch.cuda.synchronize()
    single_ms = e0.elapsed_time(e1)
    ref_l = ref.l
    ref.close()
    out = {"config": a.config, "events": n, "single_engine_ms": single_ms, "runs": []}
    print(json.dumps({"single_engine_ms": single_ms}), flush=True)
    for B in [int(v) for v in a.batch.split(",")]:
        for world in [int(v) for v in a.bands.split(",")]:
            for G0 in [int(v) for v in a.halo.split(",")]:
                G = bands.halo_rows_for(geom.height, world, G0)
                engines = [ReconstructionEngine(geom, params, halo_band=(y0, y0 + r, G), batch_capacity=B)
                           for y0, r in bands.band_rows(geom.height, world)]
                busy = np.zeros((world,), np.float64)
                per_batch = []
                rounds = []
                wrapped = []
                for r_, e in enumerate(engines):
                    wrapped.append(_Timed(e))
                for rep in range(2):   # second pass timed (first warms the engines up)
                    for w in wrapped:
                        w.e.reset()
                    per_batch.clear()
                    rounds.clear()
                    for s in range(0, n, B):
                        for w in wrapped:
                            w.clear()
                        rounds.append(bands.run_local_halo_bands(wrapped, DeviceEventArray(xd[s:s + B], yd[s:s + B],
                                                                                         pd[s:s + B])))
                        torch.cuda.synchronize()
                        per_batch.append([w.ms() for w in wrapped])
                pb = np.array(per_batch)
                busy = pb.sum(0)
                full = np.concatenate([e.l.reshape(geom.height, geom.width)[y0:y0 + r]
                                       for e, (y0, r) in zip(engines, bands.band_rows(geom.height, world))])
                exact = bool(np.array_equal(full.reshape(-1), ref_l))
                row = {"bands": world, "halo": G, "batch": B, "exact": exact,
                       "rounds_mean": float(np.mean(rounds)), "rounds_max": int(max(rounds)),
                       "projected_ms": float(pb.max(1).sum()), "busy_ms_per_rank": [round(v, 2) for v in busy],
                       "round_trips": int(sum(rounds))}
                out["runs"].append(row)
                print(json.dumps(row), flush=True)
                for e in engines:
                    e.close()
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


class _Timed:
    """Brackets an engine's halo calls with CUDA events (per-rank busy time)."""

    def __init__(self, e):
        import torch
        self.e = e
        self.device = e.device
        self._torch = torch
        self.ev = []

    def clear(self):
        self.ev = []

    def _wrap(self, fn, *args):
        t = self._torch.cuda
        a, b = t.Event(enable_timing=True), t.Event(enable_timing=True)
        a.record()
        r = fn(*args)
        b.record()
        self.ev.append((a, b))
        return r

    def halo_batch(self, blk):
        return self._wrap(self.e.halo_batch, blk)

    def halo_round(self, rnd, i, o):
        return self._wrap(self.e.halo_round, rnd, i, o)

    def halo_finish(self):
        return self._wrap(self.e.halo_finish)

    def ms(self):
        return sum(a.elapsed_time(b) for a, b in self.ev)


if __name__ == "__main__":
    main()
