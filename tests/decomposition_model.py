"""Executable model of the CUDA decomposition (test infrastructure only).

This is NOT a product path: it is a slow, loop-by-loop Python statement of the
exact data flow the CUDA kernels in paper_2510_20071_b200/csrc implement, so
the *algorithm* (links, speculative window pass, stale list, blur dependency
rules, final pass) can be checked against the oracle on the CPU, in seconds,
before any GPU time is spent.  Array names follow the kernels:

  link      : per sorted position -> dp[jj] = (j - prev_pix, j - prev_tile),
              ring rnext[k] = (next_pix - k, next_tile - k), PT[c] = (st, len)
  window    : s_j for every event (exactly the reference's FIFO)
  stale     : popped k in [s_start, s_end), stale iff next_pix(k) > popj(k)
  temporal  : per pixel segment, p_bar chain, t2 = h*d (per event), L0 chain
  blur      : blur item p (k = s_start + p) reads each tap's value at its time
  final     : l at batch end per touched pixel, last-touch update
"""

from __future__ import annotations

import numpy as np

INF = 0xFFFFFFFF
f32 = np.float32


class DecompositionModel:
    def __init__(self, width, height, params, *, gain=None, regulate_every=1, blur_enabled=True,
                 batch_cap=1 << 16, chunk=64, warm=64):
        self.W, self.H = width, height
        n = width * height
        self.n = n
        self.ts = params.tile_side
        self.A = self.ts * self.ts
        self.tx = -(-width // self.ts)
        self.ty = -(-height // self.ts)
        self.params = params
        self.every = regulate_every
        self.blur_on = blur_enabled
        self.spatial = params.spatial_enabled
        self.num, self.den = params.fill_ratio_target.numerator, params.fill_ratio_target.denominator
        self.qmin, self.qmax = params.q_min, params.q_max
        self.alpha = f32(params.alpha)
        self.oma = f32(1.0 - params.alpha)
        self.beta = f32(params.beta)
        self.h = f32(params.half_one_plus_beta)
        self.gain = None if gain is None else np.asarray(gain, np.float32).reshape(-1)
        self.pbar = np.zeros(n, np.float32)
        self.l = np.zeros(n, np.float32)
        self.last_pix = np.full(n, -1, np.int64)
        self.last_tile = np.full(self.tx * self.ty, -1, np.int64)
        self.bcap = batch_cap
        self.R = n + 1 + batch_cap
        self.rkey = np.zeros(self.R, np.int64)
        self.rnp = np.full(self.R, INF, np.int64)
        self.rnt = np.full(self.R, INF, np.int64)
        self.E = 0
        self.s = 0
        q0 = min(max(n // 16, self.qmin), self.qmax)
        self.q = q0
        self.qtmin = self.qtmax = q0
        self.npix = self.ntiles = 0
        self.evctr = 0
        self.blurs = self.stales = 0
        self.chunk, self.warm = chunk, warm
        self.spec_mismatch = 0
        self.spec_chunks = 0
        self.stale_k_log, self.stale_j_log = [], []

    # -- helpers ------------------------------------------------------------
    def _target(self, ln, npix, ntiles):
        qn = (ln * self.num * ntiles * self.A) // (self.den * npix)
        return min(max(qn, self.qmin), self.qmax)

    def _run_window(self, E0, B, dp, state, j_from, j_to, S=None):
        """Serial window recurrence from `state` (after event j_from-1) through j_to-1."""
        s, q, npix, ntiles, evctr, qtmin, qtmax = state
        for j in range(j_from, j_to):
            dpp, dpt = dp[j - E0]
            npix += dpp > j - s
            ntiles += dpt > j - s
            while j - s + 1 > q:
                k = s
                r = k % self.R
                if self.rnp[r] > j - k:
                    npix -= 1
                if self.rnt[r] > j - k:
                    ntiles -= 1
                s += 1
            evctr += 1
            if evctr >= self.every:
                evctr = 0
                if npix >= 1 and ntiles >= 1:
                    q = self._target(j - s + 1, npix, ntiles)
                    qtmin, qtmax = min(qtmin, q), max(qtmax, q)
            if S is not None:
                S[j - E0] = s
        return (s, q, npix, ntiles, evctr, qtmin, qtmax)

    def _anchor_counts(self, E0, dp, s0, j0, npix0, ntiles0, s1, j1):
        """Exact distinct counts for window [s1, j1] from those of [s0, j0] (s0<=s1, j0<=j1)."""
        npix, ntiles = npix0, ntiles0
        for k in range(j0 + 1, j1 + 1):          # grow the right edge with start s0
            dpp, dpt = dp[k - E0]
            npix += dpp > k - s0
            ntiles += dpt > k - s0
        for k in range(s0, s1):                  # shrink the left edge at end j1
            r = k % self.R
            npix -= self.rnp[r] > j1 - k
            ntiles -= self.rnt[r] > j1 - k
        return npix, ntiles

    def _speculative_window(self, E0, B, dp, state0):
        """Chunked speculation + serial verify/fix; returns S and the final state."""
        C, Wm = self.chunk, self.warm
        T = -(-B // C)
        S = np.zeros(B, np.int64)
        q_guess = state0[1]
        # anchors: state after event a_c - 1, guessed window [s'_c, a_c - 1]
        anchors = []
        prev = (state0[0], E0 - 1, state0[2], state0[3])
        for c in range(T):
            b = E0 + c * C
            if c == 0:
                anchors.append((state0[0], E0, state0[2], state0[3]))
                continue
            a = max(E0, b - Wm)
            sg = max(prev[0], a - q_guess)
            npx, ntl = self._anchor_counts(E0, dp, prev[0], prev[1], prev[2], prev[3], sg, a - 1)
            prev = (sg, a - 1, npx, ntl)
            anchors.append((sg, a, npx, ntl))
        starts, ends, outs = [], [], []
        for c in range(T):
            b = E0 + c * C
            e = min(E0 + B, b + C)
            sg, a, npx, ntl = anchors[c]
            if c == 0:
                st = state0
            else:
                # evctr and the q extrema are exact functions of j / reductions; q is guessed
                st = (sg, q_guess, npx, ntl, (state0[4] + (a - E0)) % self.every, 1 << 62, -1)
                st = self._run_window(E0, B, dp, st, a, b)
            starts.append(st)
            Sc = np.zeros(B, np.int64)
            en = self._run_window(E0, B, dp, (st[0], st[1], st[2], st[3], st[4], 1 << 62, -1), b, e, Sc)
            outs.append(Sc[b - E0:e - E0])
            ends.append(en)
        # verify / fix serially
        qtmin, qtmax = state0[5], state0[6]
        cur = state0
        for c in range(T):
            b = E0 + c * C
            e = min(E0 + B, b + C)
            self.spec_chunks += 1
            if c > 0 and (starts[c][0], starts[c][1]) != (cur[0], cur[1]):
                self.spec_mismatch += 1
                Sc = np.zeros(B, np.int64)
                en = self._run_window(E0, B, dp, (cur[0], cur[1], cur[2], cur[3], cur[4], 1 << 62, -1), b, e, Sc)
                outs[c] = Sc[b - E0:e - E0]
                ends[c] = en
            en = ends[c]
            S[b - E0:e - E0] = outs[c]
            qtmin, qtmax = min(qtmin, en[5]), max(qtmax, en[6])
            cur = (en[0], en[1], en[2], en[3], en[4], qtmin, qtmax)
        return S, cur

    # -- one device batch ----------------------------------------------------
    def process(self, x, y, p, speculative=True):
        x = np.asarray(x, np.int64)
        y = np.asarray(y, np.int64)
        keep = (x < self.W) & (y < self.H)
        x, y, p = x[keep], y[keep], np.asarray(p)[keep]
        B = len(x)
        if B == 0:
            return
        assert B <= self.bcap
        E0 = self.E
        key = y * self.W + x
        tile = (y // self.ts) * self.tx + x // self.ts
        tkey = tile * self.A + (y % self.ts) * self.ts + (x % self.ts)
        order = np.argsort(tkey, kind="stable")          # stable radix sort by tile-major key
        skey, sidx = tkey[order], order
        spix = key[order]
        stile = tile[order]
        # ---- link -----------------------------------------------------------
        dp = np.zeros((B, 2), np.int64)
        PT_st, PT_len = {}, {}
        seg_bounds = []
        i = 0
        while i < B:
            jn = i
            while jn < B and skey[jn] == skey[i]:
                jn += 1
            seg_bounds.append((i, jn))
            PT_st[int(spix[i])] = i
            PT_len[int(spix[i])] = jn - i
            i = jn
        tile_bounds = {}
        for (a, b) in seg_bounds:
            t = int(stile[a])
            lo, hi = tile_bounds.get(t, (a, b))
            tile_bounds[t] = (min(lo, a), max(hi, b))
        for (a, b) in seg_bounds:
            c = int(spix[a])
            t = int(stile[a])
            ta, tb = tile_bounds[t]
            tj = sidx[ta:tb]
            for i in range(a, b):
                jj = int(sidx[i])
                j = E0 + jj
                prev_p = E0 + int(sidx[i - 1]) if i > a else int(self.last_pix[c])
                next_p = E0 + int(sidx[i + 1]) if i + 1 < b else None
                earlier = tj[tj < jj]
                later = tj[tj > jj]
                prev_t = E0 + int(earlier.max()) if earlier.size else int(self.last_tile[t])
                next_t = E0 + int(later.min()) if later.size else None
                dp[jj, 0] = INF if prev_p < 0 else min(j - prev_p, INF)
                dp[jj, 1] = INF if prev_t < 0 else min(j - prev_t, INF)
                r = j % self.R
                self.rkey[r] = c
                self.rnp[r] = INF if next_p is None else next_p - j
                self.rnt[r] = INF if next_t is None else next_t - j
                if i == a and prev_p >= max(0, E0 + B - self.R):
                    self.rnp[prev_p % self.R] = j - prev_p
                if not earlier.size and prev_t >= max(0, E0 + B - self.R):
                    self.rnt[prev_t % self.R] = j - prev_t
        # ---- temporal -----------------------------------------------------------
        t2 = np.zeros(B, np.float32)
        L0 = np.zeros(B, np.float32)
        for (a, b) in seg_bounds:
            c = int(spix[a])
            pb = self.pbar[c]
            lv = self.l[c]
            for i in range(a, b):
                pol = f32(p[sidx[i]])
                pb = f32(f32(self.alpha * pb) + f32(self.oma * pol))
                d = f32(pol - pb)
                if self.gain is not None:
                    d = f32(d * self.gain[c])
                t2[i] = f32(self.h * d)
                lv = f32(f32(self.beta * lv) + t2[i])
                L0[i] = lv
            self.pbar[c] = pb
            if not self.spatial:
                self.l[c] = lv
        if not self.spatial:
            for (a, b) in seg_bounds:
                self.last_pix[int(spix[a])] = E0 + int(sidx[b - 1])
            self.E += B
            return
        # ---- window -----------------------------------------------------------
        state0 = (self.s, self.q, self.npix, self.ntiles, self.evctr, self.qtmin, self.qtmax)
        if speculative:
            S, fin = self._speculative_window(E0, B, dp, state0)
            S_ref = np.zeros(B, np.int64)
            fin_ref = self._run_window(E0, B, dp, state0, E0, E0 + B, S_ref)
            assert np.array_equal(S, S_ref) and fin[:5] == fin_ref[:5], "speculation diverged"
            assert fin[5:] == fin_ref[5:]
        else:
            S = np.zeros(B, np.int64)
            fin = self._run_window(E0, B, dp, state0, E0, E0 + B, S)
        s_start, s_end = self.s, int(fin[0])
        # ---- stale list -------------------------------------------------------
        npop = s_end - s_start
        popj = np.zeros(npop, np.int64)
        prev_s = s_start
        for jj in range(B):
            for k in range(prev_s, int(S[jj])):
                popj[k - s_start] = E0 + jj
            prev_s = int(S[jj])
        stale = np.array([self.rnp[(s_start + q) % self.R] > popj[q] - (s_start + q) for q in range(npop)], bool)
        self.stale_k_log.append(s_start + np.nonzero(stale)[0])
        self.stale_j_log.append(popj[stale])
        nst = int(stale.sum())
        self.stales += nst
        # ---- blur -------------------------------------------------------------
        Bval = {}

        def is_blurred(e):          # event e (global) has a blur in this batch -> its item index
            if s_start <= e < s_end and stale[e - s_start]:
                return e - s_start
            return None

        def value_after(c, i_pos, a):
            """l of pixel c right after the temporal update at sorted position i_pos (segment start a)."""
            pos = i_pos - 1
            while pos >= a:
                bi = is_blurred(E0 + int(sidx[pos]))
                if bi is not None:
                    v = Bval[bi]
                    break
                pos -= 1
            else:
                lp = int(self.last_pix[c])
                bi = is_blurred(lp) if lp >= 0 else None
                if bi is None:
                    return L0[i_pos]
                v = Bval[bi]
            for q2 in range(pos + 1, i_pos + 1):
                v = f32(f32(self.beta * v) + t2[q2])
            return v

        def tapval(n_, J, pb_):
            a = PT_st.get(n_)
            lp = int(self.last_pix[n_])
            carried = is_blurred(lp) if lp >= 0 else None
            if a is None or E0 + int(sidx[a]) > J:
                if carried is not None and carried < pb_:
                    return Bval[carried]
                return self.l[n_]
            b = a + PT_len[n_]
            i_pos = a
            while i_pos + 1 < b and E0 + int(sidx[i_pos + 1]) <= J:
                i_pos += 1
            e = E0 + int(sidx[i_pos])
            bi = is_blurred(e)
            if bi is not None and bi < pb_:
                return Bval[bi]
            return value_after(n_, i_pos, a)

        if self.blur_on:
            for q2 in range(npop):
                if not stale[q2]:
                    continue
                k = s_start + q2
                c = int(self.rkey[k % self.R])
                cx, cy = c % self.W, c // self.W
                J = int(popj[q2])
                num = f32(0.0)
                den = f32(0.0)
                for dy in (-1, 0, 1):
                    yy = cy + dy
                    if yy < 0 or yy >= self.H:
                        continue
                    for dx in (-1, 0, 1):
                        xx = cx + dx
                        if xx < 0 or xx >= self.W:
                            continue
                        w = f32((2 if dy == 0 else 1) * (2 if dx == 0 else 1))
                        num = f32(num + f32(w * tapval(yy * self.W + xx, J, q2)))
                        den = f32(den + w)
                Bval[q2] = f32(num / den)
            self.blurs += nst
        # ---- final ------------------------------------------------------------
        newl = {}
        for (a, b) in seg_bounds:
            c = int(spix[a])
            bi = is_blurred(E0 + int(sidx[b - 1])) if self.blur_on else None
            newl[c] = Bval[bi] if bi is not None else (value_after(c, b - 1, a) if self.blur_on else L0[b - 1])
        if self.blur_on:
            for q2 in range(npop):
                if stale[q2]:
                    c = int(self.rkey[(s_start + q2) % self.R])
                    if c not in PT_st:
                        newl[c] = Bval[q2]
        for c, v in newl.items():
            self.l[c] = v
        for (a, b) in seg_bounds:
            c = int(spix[a])
            self.last_pix[c] = E0 + int(sidx[b - 1])
        for t, (ta, tb) in tile_bounds.items():
            self.last_tile[t] = E0 + int(sidx[ta:tb].max())
        self.s, self.q, self.npix, self.ntiles, self.evctr, self.qtmin, self.qtmax = fin
        self.E += B

    # -- reference-layout views ------------------------------------------------
    def qs(self):
        head = self.s % (self.n + 1)
        return np.array([head, self.E - self.s, self.q, self.npix, self.ntiles, self.blurs, self.stales,
                         self.qtmin, self.qtmax, self.evctr], np.int64)

    def active_count(self):
        cnt = np.zeros(self.n, np.int64)
        for k in range(self.s, self.E):
            cnt[self.rkey[k % self.R]] += 1
        return np.minimum(cnt, 65535).astype(np.uint16)

    def tile_count(self):
        act = self.active_count().astype(np.int64) > 0
        tc = np.zeros(self.tx * self.ty, np.int64)
        ys, xs = np.divmod(np.arange(self.n), self.W)
        np.add.at(tc, (ys // self.ts) * self.tx + xs // self.ts, act)
        return np.minimum(tc, 255).astype(np.uint8)

    def ring_xy(self):
        qcap = self.n + 1
        qx = np.zeros(qcap, np.uint16)
        qy = np.zeros(qcap, np.uint16)
        for k in range(max(0, self.E - qcap), self.E):
            c = self.rkey[k % self.R]
            qx[k % qcap] = c % self.W
            qy[k % qcap] = c // self.W
        return qx, qy
