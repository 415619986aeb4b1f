"""CPU stand-in for a halo-band engine (filter-ON row bands), test infrastructure.

It exposes the same halo protocol as the native engine
(``halo_batch`` / ``halo_round`` / ``halo_finish``) so the
world-size-2 gloo test can run ``bands.HaloBandEngine``'s exchange logic on
the CPU.  The global stale schedule comes from the C oracle run on the whole
stream (every rank sees every event); the band's rows are then replayed in
Python float32 in the reference's order (_kernels.py:120-189): temporal update
of the event's pixel, then the blurs popped at that event in pop order.  Items
of the outermost halo rows take the neighbours' values; every value carries a
taint bit (it read a halo value that was not final).  Each round replays the
whole batch from its starting state; the native engine only re-runs tainted
items, which gives the same values and taints (taints only ever clear).
"""

from __future__ import annotations

import numpy as np

F32 = np.float32
_W9 = [F32((1 if dy != 0 else 2) * (1 if dx != 0 else 2)) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]


class HaloOracleBand:
    def __init__(self, geom, params, *, halo_band, batch_capacity=None):
        from oracle import oracle as orc
        self.W, self.H = geom.width, geom.height
        self.y0, self.y1, G = halo_band
        self.reg0, self.reg1 = max(0, self.y0 - G), min(self.H, self.y1 + G)
        self.in_rows = (self.y0 - G if self.y0 > 0 else -1, self.y1 + G - 1 if self.y1 < self.H else -1)
        self.out_rows = (self.y0 + G - 1 if self.y0 > 0 else -1, self.y1 - G if self.y1 < self.H else -1)
        self.win = orc.OracleEngine(self.W, self.H, params, record_stale=True)
        n = self.W * self.H
        self.l = np.zeros(n, F32)
        self.p_bar = np.zeros(n, F32)
        self.a, self.oma = F32(params.alpha), F32(1.0 - params.alpha)
        self.b, self.h = F32(params.beta), F32(params.half_one_plus_beta)
        self.pix = np.zeros(0, np.int64)    # pixel of every in-bounds event so far
        self.E = 0
        self.oob = 0

    # -- protocol ---------------------------------------------------------------
    def halo_batch(self, blk):
        x = np.asarray(blk.x, np.int64)
        y = np.asarray(blk.y, np.int64)
        keep = (x < self.W) & (y < self.H)
        self.oob += int((~keep).sum())
        nk = len(self.win.stale_k)
        self.win.process_array(blk.t, blk.x, blk.y, blk.p)
        sk = self.win.stale_k[nk] if len(self.win.stale_k) > nk else np.zeros(0, np.int64)
        sj = self.win.stale_j[nk] if len(self.win.stale_j) > nk else np.zeros(0, np.int64)
        self.bx = (y[keep] * self.W + x[keep])
        self.bp = np.asarray(blk.p, np.int8)[keep]
        self.pix = np.concatenate([self.pix, self.bx])
        self.items = [(int(j) - self.E, int(self.pix[k])) for k, j in zip(sk, sj)]
        rows = [c // self.W for _, c in self.items]
        self.lists = [[i for i, r in enumerate(rows) if r == want] for want in self.in_rows + self.out_rows]
        self.slot = {}
        for s, i in enumerate(self.lists[0] + self.lists[1]):
            self.slot[i] = s
        self.l0, self.pb0 = self.l.copy(), self.p_bar.copy()
        return tuple(len(v) for v in self.lists)

    def halo_round(self, rnd, recv, send):
        words = recv.numpy() if hasattr(recv, "numpy") else np.asarray(recv)
        l, pb = self.l0.copy(), self.pb0.copy()
        taint = np.zeros(len(l), bool)
        vals, tnts = np.zeros(len(self.items), F32), np.zeros(len(self.items), bool)
        W, H = self.W, self.H
        it = 0
        for j in range(len(self.bx)):
            c = int(self.bx[j])
            if self.reg0 <= c // W < self.reg1:
                p = F32(self.bp[j])
                v = self.a * pb[c] + self.oma * p
                pb[c] = v
                d = p - v
                l[c] = self.b * l[c] + self.h * d
            while it < len(self.items) and self.items[it][0] == j:
                c = self.items[it][1]
                cy, cx = divmod(c, W)
                if self.reg0 <= cy < self.reg1:
                    if cy in self.in_rows:
                        w = int(words[self.slot[it]])
                        v = np.array([w & 0xFFFFFFFF], np.uint32).view(F32)[0]
                        t = w < 0
                    else:
                        num, den, t = F32(0), F32(0), False
                        for q in range(9):
                            yy, xx = cy + q // 3 - 1, cx + q % 3 - 1
                            if 0 <= yy < H and 0 <= xx < W:
                                num = num + _W9[q] * l[yy * W + xx]
                                den = den + _W9[q]
                                t = t or bool(taint[yy * W + xx])
                        v = num / den
                    l[c] = v
                    taint[c] = t
                    vals[it], tnts[it] = v, t
                it += 1
        out = self.lists[2] + self.lists[3]
        o = np.array([int(vals[i:i + 1].view(np.uint32)[0]) | ((1 << 63) if tnts[i] else 0) for i in out],
                     np.uint64).view(np.int64)
        if len(o):
            import torch
            send.copy_(torch.from_numpy(o))
        self._l, self._pb = l, pb

    def halo_finish(self):
        self.l, self.p_bar = self._l, self._pb
        self.E += len(self.bx)

    def _counters(self):
        return self.E, self.oob
