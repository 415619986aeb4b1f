"""Filter-ON row bands: how many halo-exchange rounds does a batch need?

Analysis tool (CPU, numba), not on the product path.  For a stream and its
global stale schedule (the C oracle's stale log), simulate the round
structure of the banded filter-ON engine without the floats:
rank r computes the items of rows (y0 - G, y1 + G - 1), takes the items of its
halo rows y0 - G / y1 + G - 1 from their owners, and an item computed in
round k is exact iff every value it read was exact.  R_r(p) = the first round
in which rank r's value of item p is exact; an injected item is exact one
round after its owner's.  A batch needs max_injected R_owner(p) + 1 rounds
(the last one re-runs with all-exact halo inputs).

    python scripts/band_rounds.py --config 2 --events 3000000 --bands 2,4,8 --halo 1,4,8
"""

from __future__ import annotations

import argparse
import os
import sys
from fractions import Fraction

import numpy as np
import numba

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


@numba.njit(cache=True)
def rounds_per_batch(px, sk, sj, W, H, E, batch, y0s, y1s, G):
    """px: pixel of every in-bounds event; (sk, sj): stale log in pop order."""
    nb = (E + batch - 1) // batch
    N = len(y0s)
    out = np.ones(nb, np.int64)
    pixR = np.zeros((N, W * H), np.int64)   # round in which rank r's current value of the pixel is exact
    touched = np.zeros((N, W * H), np.uint8)
    owner = np.empty(H, np.int64)
    for r in range(N):
        for y in range(y0s[r], y1s[r]):
            owner[y] = r
    ns = len(sk)
    i = 0
    for b in range(nb):
        e0 = b * batch
        e1 = min(E, e0 + batch)
        for r in range(N):
            pixR[r, :] = 1
        mx = 0
        while i < ns and sj[i] < e1:
            c = px[sk[i]]
            cy = c // W
            cx = c - cy * W
            # owner first: its value of the item
            o = owner[cy]
            Ro = 1
            for dy in range(-1, 2):
                yy = cy + dy
                if yy < 0 or yy >= H:
                    continue
                for dx in range(-1, 2):
                    xx = cx + dx
                    if xx < 0 or xx >= W:
                        continue
                    v = pixR[o, yy * W + xx]
                    if v > Ro:
                        Ro = v
            for r in range(N):
                lo = max(0, y0s[r] - G)
                hi = min(H, y1s[r] + G)
                if cy < lo or cy >= hi:
                    continue
                inj = (cy == y0s[r] - G and y0s[r] > 0) or (cy == y1s[r] + G - 1 and y1s[r] < H)
                if r == o:
                    pixR[r, c] = Ro
                elif not inj:
                    R = 1
                    for dy in range(-1, 2):
                        yy = cy + dy
                        if yy < 0 or yy >= H:
                            continue
                        for dx in range(-1, 2):
                            xx = cx + dx
                            if xx < 0 or xx >= W:
                                continue
                            v = pixR[r, yy * W + xx]
                            if v > R:
                                R = v
                    pixR[r, c] = R
                if inj:
                    pixR[r, c] = Ro + 1
                    if Ro > mx:
                        mx = Ro
            i += 1
        out[b] = mx + 1 if mx > 0 else 1
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--events", type=int, default=3_000_000)
    ap.add_argument("--batch", type=int, default=1 << 20)
    ap.add_argument("--bands", default="2,4,8")
    ap.add_argument("--halo", default="1,2,4,8")
    a = ap.parse_args()
    from oracle import oracle as orc
    from paper_2510_20071_b200 import workloads
    from paper_2510_20071_b200.core import SensorGeometry, compute_params
    W, H = {2: (640, 480), 3: (1280, 720), 5: (2560, 1440)}[a.config]
    if a.config == 3:
        ev = workloads.texture_noise_hot(W, H, a.events, seed=0)
    else:
        ev = workloads.moving_texture(W, H, a.events, seed=0, speed=1000.0 if a.config == 5 else 200.0)
    geom = SensorGeometry(W, H)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=True)
    ref = orc.OracleEngine(W, H, params, record_stale=True)
    for s in range(0, len(ev), 1 << 20):
        blk = ev.slice(s, s + (1 << 20))
        ref.process_array(blk.t, blk.x, blk.y, blk.p)
    sk, sj = ref.stale_log()
    px = ev.y.astype(np.int64) * W + ev.x.astype(np.int64)
    from paper_2510_20071_b200 import bands
    for N in [int(v) for v in a.bands.split(",")]:
        br = bands.band_rows(H, N)
        y0s = np.array([y0 for y0, _ in br], np.int64)
        y1s = np.array([y0 + r for y0, r in br], np.int64)
        for G in [int(v) for v in a.halo.split(",")]:
            rr = rounds_per_batch(px, sk, sj, W, H, len(px), a.batch, y0s, y1s, G)
            print(f"config {a.config} bands {N} halo {G}: rounds per batch {rr.tolist()} (mean {rr.mean():.1f})",
                  flush=True)


if __name__ == "__main__":
    main()
