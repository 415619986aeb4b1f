// fibar_front.cu -- the front end of a device batch: ingest (OOB filter, compaction),
// pixel/tile links, the exact window pass (speculation + verification) and the
// eviction pass (stale items).  See fibar_engine.cu for the batch flow.
#include "fibar_kernels.cuh"

namespace fibar {

static __constant__ long long c_fine_mul[NFINE] = {-8, -4, -2, -1, 0, 1, 2, 4, 8, 16};
static __constant__ long long c_lin_off[NLIN] = {-16384, -4096, -1024, 0, 1024, 4096, 16384};
static __constant__ double c_geo_mul[NGEO] = {0.25, 0.5, 0.75, 1.25, 1.5, 2.0, 2.5, 3.0, 4.0, 6.0, 8.0, 12.0};

// ---------------------------------------------------------------- ingest ---


// an event is kept iff it lies on the sensor (else it is out of bounds,
// counted like pipeline.py:209-210) and in this engine's row band (a band
// engine silently leaves other bands' events to their owners)
__device__ __forceinline__ bool on_sensor(const Ctx &x, unsigned xx, unsigned yy) {
  return xx < (unsigned)x.W && yy < x.full_H;
}
__device__ __forceinline__ bool in_band(const Ctx &x, unsigned yy) { return yy - x.band_y0 < (unsigned)x.H; }

// a thread's IN_ITEMS consecutive packet entries: one 16-byte load per
// coordinate column and one 8-byte load of polarities when the packet is
// aligned (lanes take consecutive 16-byte pieces: coalesced), else scalar
__device__ __forceinline__ long long raw_count(const Ctx &x) { return x.n_raw_dev ? *x.n_raw_dev : x.n_raw; }

__device__ __forceinline__ void load_in(const Ctx &x, long long n_raw, long long base, unsigned (&xx)[IN_ITEMS],
                                        unsigned (&yy)[IN_ITEMS], int (&pp)[IN_ITEMS], bool with_p) {
  static_assert(IN_ITEMS == 8, "vector ingest assumes 8 entries per thread");
  const bool vec = base + IN_ITEMS <= n_raw && ((reinterpret_cast<uintptr_t>(x.raw_x + base) |
                                                   reinterpret_cast<uintptr_t>(x.raw_y + base)) & 15) == 0 &&
                   (!with_p || (reinterpret_cast<uintptr_t>(x.raw_p + base) & 7) == 0);
  if (vec) {
    const uint4 vx = *reinterpret_cast<const uint4 *>(x.raw_x + base);
    const uint4 vy = *reinterpret_cast<const uint4 *>(x.raw_y + base);
    const unsigned wx[4] = {vx.x, vx.y, vx.z, vx.w}, wy[4] = {vy.x, vy.y, vy.z, vy.w};
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      xx[2 * r] = wx[r] & 0xFFFFu;
      xx[2 * r + 1] = wx[r] >> 16;
      yy[2 * r] = wy[r] & 0xFFFFu;
      yy[2 * r + 1] = wy[r] >> 16;
    }
    if (with_p) {
      const uint2 vp = *reinterpret_cast<const uint2 *>(x.raw_p + base);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        pp[r] = (int)(int8_t)(vp.x >> (8 * r));
        pp[4 + r] = (int)(int8_t)(vp.y >> (8 * r));
      }
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < IN_ITEMS; ++r) {
    const long long i = base + r;
    const bool in = i < n_raw;
    xx[r] = in ? x.raw_x[i] : 0xFFFFu;   // off the sensor: never kept
    yy[r] = in ? x.raw_y[i] : 0xFFFFu;
    if (with_p) pp[r] = in ? x.raw_p[i] : 0;
  }
}

__global__ void __launch_bounds__(TPB) k_count_inb(Ctx x, int nblocks) {
  pdl_wait();
  __shared__ unsigned wsum[TPB / 32], woob[TPB / 32];
  const long long base = (long long)blockIdx.x * IN_TILE + threadIdx.x * IN_ITEMS;
  unsigned cnt = 0, oob = 0;
  const long long n_raw = raw_count(x);
  unsigned xs[IN_ITEMS], ys[IN_ITEMS];
  int ps[IN_ITEMS];
  load_in(x, n_raw, base, xs, ys, ps, false);
#pragma unroll
  for (int r = 0; r < IN_ITEMS; ++r) {
    if (base + r < n_raw) {
      const bool ok = on_sensor(x, xs[r], ys[r]);
      oob += !ok;
      cnt += ok && in_band(x, ys[r]);
    }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  oob = __reduce_add_sync(0xffffffffu, oob);
  if ((threadIdx.x & 31) == 0) {
    wsum[threadIdx.x >> 5] = cnt;
    woob[threadIdx.x >> 5] = oob;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0, o = 0;
    for (int w = 0; w < TPB / 32; ++w) {
      t += wsum[w];
      o += woob[w];
    }
    x.blockcnt[blockIdx.x] = t;
    if (blockIdx.x == 0) x.blockcnt[nblocks] = 0;
    if (o) atomicAdd((unsigned long long *)&x.st->oob, (unsigned long long)o);
  }
}

__device__ __forceinline__ void open_batch(const Ctx &x);

// fused != 0 (one block only): the packet fits one tile, so the block also
// counts the out-of-bounds events and takes its total from its own scan --
// no k_count_inb, no scan kernel
__global__ void __launch_bounds__(TPB) k_compact(Ctx x, int nblocks, int fused) {
  pdl_wait();
  __shared__ unsigned wsum[TPB / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long base = (long long)blockIdx.x * IN_TILE + threadIdx.x * IN_ITEMS;
  bool keep[IN_ITEMS];
  unsigned cnt = 0;
  const long long n_raw = raw_count(x);
  unsigned xs[IN_ITEMS], ys[IN_ITEMS];
  int ps[IN_ITEMS];
  load_in(x, n_raw, base, xs, ys, ps, true);
#pragma unroll
  unsigned oob = 0;
  for (int r = 0; r < IN_ITEMS; ++r) {
    const bool ok = base + r < n_raw && on_sensor(x, xs[r], ys[r]);
    oob += (fused && base + r < n_raw && !ok) ? 1u : 0u;
    keep[r] = ok && in_band(x, ys[r]);
    cnt += keep[r];
  }
  if (fused) {
    oob = __reduce_add_sync(0xffffffffu, oob);
    if (lane == 0 && oob) atomicAdd((unsigned long long *)&x.st->oob, (unsigned long long)oob);
  }
  unsigned incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  unsigned wofs = 0;
  for (int w = 0; w < wid; ++w) wofs += wsum[w];
  unsigned pos = (fused ? 0u : x.blockcnt[blockIdx.x]) + wofs + incl - cnt;
#pragma unroll
  for (int r = 0; r < IN_ITEMS; ++r) {
    if (!keep[r]) continue;
    const unsigned xx = xs[r], yy = ys[r] - x.band_y0;
    const unsigned key = yy * (unsigned)x.W + xx;
    const unsigned tile = (yy / x.ts) * (unsigned)x.tiles_x + xx / x.ts;
    const unsigned sub = (yy % x.ts) * x.ts + xx % x.ts;
    x.ekey[pos] = key;
    x.tkey[pos] = tile * (unsigned)x.A + sub;
    x.epol[pos] = (int8_t)ps[r];
    ++pos;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // the batch's own scalars; what depends on the window state (E0, s_start,
    // epoch) is set by k_batch_begin, so ingest may run ahead of the previous
    // batch's window pass
    BatchState *b = x.bs;
    unsigned total = 0;
    if (fused)
      for (int w = 0; w < TPB / 32; ++w) total += wsum[w];
    b->B = fused ? total : x.blockcnt[nblocks];
    b->npop = 0;
    b->stale_batch = 0;
    b->ticket = 0;
    b->nlong = 0;
    b->nco = 0;
    b->nbad = 0;
    b->vcnt[0] = 0;
    b->vcnt[1] = 0;
    b->qlo = 0x7FFFFFFFFFFFFFFFLL;
    b->qhi = -1;
    b->nclosed = 0;
    if (!x.spatial) {
      // filter OFF runs on one stream, batch after batch: the batch's first
      // event index, its opening and its event count need no kernels of their
      // own (filter ON: k_ingest_end in batch order, k_window_run, k_posinfo)
      DevState *s = x.st;
      b->E0 = s->Ein;
      s->Ein += b->B;
      open_batch(x);
      s->E += b->B;
    }
  }
}

// A small batch's packet into the fixed input buffers its captured ingest
// graph reads, with the batch's raw count (graphs are captured per size class,
// sized for the class's upper bound, and read the real count here).
__global__ void __launch_bounds__(TPB) k_stage(const uint16_t *sx, const uint16_t *sy, const int8_t *sp, long long n,
                                               uint16_t *dx, uint16_t *dy, int8_t *dp, long long *n_dev) {
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_dev = n;
  const bool vec = ((reinterpret_cast<uintptr_t>(sx) | reinterpret_cast<uintptr_t>(sy)) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(sp) & 7) == 0;
  const long long stride = (long long)gridDim.x * TPB;
  long long i0 = 0;
  if (vec) {
    const long long nv = n / 8;
    for (long long v = (long long)blockIdx.x * TPB + threadIdx.x; v < nv; v += stride) {
      reinterpret_cast<uint4 *>(dx)[v] = reinterpret_cast<const uint4 *>(sx)[v];
      reinterpret_cast<uint4 *>(dy)[v] = reinterpret_cast<const uint4 *>(sy)[v];
      reinterpret_cast<uint2 *>(dp)[v] = reinterpret_cast<const uint2 *>(sp)[v];
    }
    i0 = nv * 8;
  }
  for (long long i = i0 + (long long)blockIdx.x * TPB + threadIdx.x; i < n; i += stride) {
    dx[i] = sx[i];
    dy[i] = sy[i];
    dp[i] = sp[i];
  }
}

// Non-contiguous device packets into the device staging set: one CTA per
// packet (grid-stride within it), 16-byte vector copies when the source and
// destination line up, element copies otherwise.
__global__ void __launch_bounds__(TPB) k_gather(const GatherTable tab, uint16_t *dx, uint16_t *dy, int8_t *dp) {
  pdl_wait();
  // packet blockIdx.y, split over gridDim.x CTAs in contiguous pieces
  const GatherEntry ef = tab.e[blockIdx.y];
  const long long per = (ef.n + gridDim.x - 1) / gridDim.x;
  const long long p0 = min(ef.n, (long long)blockIdx.x * ((per + 7) & ~7LL));
  const long long p1 = min(ef.n, p0 + ((per + 7) & ~7LL));
  GatherEntry e = ef;
  e.x += p0;
  e.y += p0;
  e.p += p0;
  e.dst += p0;
  e.n = p1 - p0;
  const bool vec = ((reinterpret_cast<uintptr_t>(e.x) | reinterpret_cast<uintptr_t>(e.y) |
                     reinterpret_cast<uintptr_t>(dx + e.dst) | reinterpret_cast<uintptr_t>(dy + e.dst)) & 15) == 0 &&
                   ((reinterpret_cast<uintptr_t>(e.p) | reinterpret_cast<uintptr_t>(dp + e.dst)) & 7) == 0;
  long long i0 = 0;
  if (vec) {
    const long long nv = e.n / 8;   // 8 events: 16 B of x, 16 B of y, 8 B of p
    for (long long v = threadIdx.x; v < nv; v += TPB) {
      reinterpret_cast<uint4 *>(dx + e.dst)[v] = reinterpret_cast<const uint4 *>(e.x)[v];
      reinterpret_cast<uint4 *>(dy + e.dst)[v] = reinterpret_cast<const uint4 *>(e.y)[v];
      reinterpret_cast<uint2 *>(dp + e.dst)[v] = reinterpret_cast<const uint2 *>(e.p)[v];
    }
    i0 = nv * 8;
  }
  for (long long i = i0 + threadIdx.x; i < e.n; i += TPB) {
    dx[e.dst + i] = e.x[i];
    dy[e.dst + i] = e.y[i];
    dp[e.dst + i] = e.p[i];
  }
}

// The batch's first event index, from the ingest's own running count (so the
// ingest, segments and links may run ahead of the previous window pass).
__global__ void k_ingest_end(Ctx x) {
  pdl_wait();
  DevState *s = x.st;
  BatchState *b = x.bs;
  b->E0 = s->Ein;
  s->Ein += b->B;
}

// Opens the batch's window part against the state the previous batch left:
// the window start and a fresh blur epoch (k_batch_begin, or the first thread
// of the front end's k_anchor).
__device__ __forceinline__ void open_batch(const Ctx &x) {
  DevState *s = x.st;
  BatchState *b = x.bs;
  b->s_start = s->s;
  s->epoch += 1;
  b->epoch = s->epoch;
  b->epoch0 = s->epoch;
}

__global__ void k_batch_begin(Ctx x) {
  pdl_wait();
  open_batch(x);
}

// ------------------------------------------------------------------ link ---

__global__ void __launch_bounds__(TPB) k_seg_marks(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const long long i = (long long)blockIdx.x * TPB + threadIdx.x;
  if (i >= B) return;
  const unsigned k = x.skey[i];
  const unsigned jj = x.sidx[i];
  const unsigned c = x.ekey[jj];
  x.rkey[(unsigned long long)(x.bs->E0 + jj) & x.Rm] = c;   // the window ring's key of event jj
  const bool head = i == 0 || x.skey[i - 1] != k;
  const bool tail = i == B - 1 || x.skey[i + 1] != k;
  if (head) x.pt[c].st = (unsigned)i;
  if (tail) x.pt[c].end = (unsigned)(i + 1);
  const unsigned t = k / x.A;
  if (i == 0 || x.skey[i - 1] / x.A != t) x.ptt[t].x = (unsigned)i;
  if (i == B - 1 || x.skey[i + 1] / x.A != t) x.ptt[t].y = (unsigned)(i + 1);
}

__global__ void __launch_bounds__(TPB) k_link(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const long long i = (long long)blockIdx.x * TPB + threadIdx.x;
  if (i >= B) return;
  const long long E0 = x.bs->E0;
  const unsigned key = x.skey[i];
  const unsigned jj = x.sidx[i];
  const long long j = E0 + jj;
  const unsigned c = x.ekey[jj];
  const unsigned t = key / x.A;
  const long long lo_ok = max(0LL, E0 + B - (long long)(x.Rm + 1));   // oldest index whose slot is not reused

  // pixel links: neighbours in the sorted order
  const bool first_pix = i == 0 || x.skey[i - 1] != key;
  const bool last_pix = i == B - 1 || x.skey[i + 1] != key;
  const long long pre_last = x.plast[c];
  const long long prev_p = first_pix ? pre_last : E0 + x.sidx[i - 1];
  const long long next_p = last_pix ? -1 : E0 + x.sidx[i + 1];

  // tile links: latest earlier / earliest later event in the tile segment
  const uint2 tr = x.ptt[t];
  long long prev_t = -1, next_t = -1;
  unsigned tmax = 0;   // the tile's latest event of the batch (its new last-touch)
  if (tr.y - tr.x <= 64) {
    unsigned best_lo = 0, best_hi = 0xFFFFFFFFu;
    bool have_lo = false;
    for (unsigned q = tr.x; q < tr.y; ++q) {
      unsigned o = x.sidx[q];
      tmax = max(tmax, o);
      if (o < jj) {
        if (!have_lo || o > best_lo) best_lo = o;
        have_lo = true;
      } else if (o > jj && o < best_hi) {
        best_hi = o;
      }
    }
    if (have_lo) prev_t = E0 + best_lo;
    if (best_hi != 0xFFFFFFFFu) next_t = E0 + best_hi;
  } else {
    const int tx = (int)(t % (unsigned)x.tiles_x), ty = (int)(t / (unsigned)x.tiles_x);
    for (int dy = 0; dy < x.ts; ++dy) {
      const int yy = ty * x.ts + dy;
      if (yy >= x.H) break;
      for (int dx = 0; dx < x.ts; ++dx) {
        const int xx = tx * x.ts + dx;
        if (xx >= x.W) break;
        const PixRec r = x.pt[(unsigned)yy * x.W + xx];
        if (r.end <= r.st) continue;
        tmax = max(tmax, x.sidx[r.end - 1]);   // a pixel's events are in stream order
        // first position in [st, end) with sidx >= jj
        unsigned lo = r.st, hi = r.end;
        while (lo < hi) {
          unsigned mid = (lo + hi) >> 1;
          if (x.sidx[mid] < jj) lo = mid + 1; else hi = mid;
        }
        if (lo > r.st) prev_t = max(prev_t, E0 + (long long)x.sidx[lo - 1]);
        unsigned up = (lo < r.end && x.sidx[lo] == jj) ? lo + 1 : lo;
        if (up < r.end) {
          long long cand = E0 + x.sidx[up];
          next_t = next_t < 0 ? cand : min(next_t, cand);
        }
      }
    }
  }
  const bool first_tile = prev_t < 0;
  if (first_tile) {
    // the tile's earliest event of the batch is the only one reading the
    // tile's last-touch; it also writes the batch's value for the next batch
    prev_t = x.last_tile[t];
    x.last_tile[t] = E0 + tmax;
  }

  x.dp[jj] = make_uint2(dist32(j, prev_p), dist32(j, prev_t));
  x.rnext[(unsigned long long)j & x.Rm] =
      make_uint2(next_p < 0 ? FIBAR_INF32 : (unsigned)(next_p - j), next_t < 0 ? FIBAR_INF32 : (unsigned)(next_t - j));
  if (first_pix) {
    // the reference's active_count saturates at 65535, after which
    // its count-based staleness departs from this exact restatement.  wcnt is
    // the pixel's exact in-window event count at batch start; the count seen
    // by its t-th event this batch is at most wcnt + t, so a batch can only
    // reach the cap if wcnt + seglen > 65535 -- flag that (never misses).
    const unsigned pend = x.pt[c].end;
    const unsigned seglen = pend - (unsigned)i;
    // (atomic: the previous batch's eviction pass may be subtracting meanwhile;
    // a count not yet decremented only makes the check more conservative)
    if (seglen > (unsigned)LONG_SEG) {   // long segment (hot pixel): listed here for k_temporal_long
      const unsigned slot = atomicAdd(&x.bs->nlong, 1u);
      if (slot < x.max_long) x.longseg[slot] = make_uint2((unsigned)i, c);
    }
    const unsigned wc = atomicAdd(&x.wcnt[c], seglen);
    if ((unsigned long long)wc + seglen > 65535ull) atomicAdd((unsigned long long *)&x.st->saturated, 1ull);
    // the pixel's last-touch for the next batch (read above by this thread
    // alone), so the next front end never waits for this batch's replay
    x.plast[c] = E0 + x.sidx[pend - 1];
  }
  if (first_pix && pre_last >= lo_ok && pre_last >= 0) {
    long long d = j - pre_last;
    x.rnext[(unsigned long long)pre_last & x.Rm].x = d >= FIBAR_INF32 ? FIBAR_INF32 : (unsigned)d;
  }
  if (first_tile && prev_t >= lo_ok && prev_t >= 0) {
    long long d = j - prev_t;
    x.rnext[(unsigned long long)prev_t & x.Rm].y = d >= FIBAR_INF32 ? FIBAR_INF32 : (unsigned)d;
  }
}

// ---------------------------------------------------------------- window ---

struct WState {
  long long s, q, npix, ntiles, evctr;
};

__device__ __forceinline__ long long chunk_warm_start(const Ctx &x, long long E0, int c) {
  return max(E0, E0 + (long long)c * x.chunk - x.warm);
}

// where chunk c's candidate windows end: its warm-up start, or for the extra
// chunk c == T (the prediction for the next batch) the batch's end
__device__ __forceinline__ long long anchor_at(const Ctx &x, long long E0, long long B, int c, int T) {
  return c < T ? chunk_warm_start(x, E0, c) : E0 + B;
}

// coarse candidate i: a dense linear grid around the batch-start target q0
// plus a geometric one that reaches windows far from it (cold start, scene change)
__device__ __forceinline__ long long cand_len(const Ctx &x, long long q0, int i) {
  long long L = i < NLIN ? q0 + c_lin_off[i] : (long long)((double)q0 * c_geo_mul[i - NLIN]);
  return L < 1 ? 1 : (L > x.qmax ? x.qmax : L);
}

// floor(N / D) for N >= 0, D > 0: a float32 reciprocal estimate (relative
// error ~1e-7, and the quotients here stay below 2^24) and an exact integer fix-up
__device__ __forceinline__ long long floordiv_nn(long long N, long long D) {
  if (N < (1LL << 53)) return (long long)floor(__ddiv_rn((double)N, (double)D));   // exact (see regulate32)
  long long q = (long long)__fmul_rn((float)N, __frcp_rn((float)D));
  if (q * D > N) {
    do { --q; } while (q * D > N);
  } else {
    while ((q + 1) * D <= N) ++q;
  }
  return q;
}

// integer fill-ratio regulation (_kernels.py:195-201)
__device__ __forceinline__ long long regulate(const Ctx &x, long long len, long long np, long long nt) {
  const long long qn = floordiv_nn(len * x.num * nt * (long long)x.A, x.den * np);
  return qn < x.qmin ? x.qmin : (qn > x.qmax ? x.qmax : qn);
}

// the same for the serial window run's 32-bit state: (len * nt) as one wide
// multiply, num * A folded on the host.  With q_max < 2^22 (every sensor up to
// 4.19M pixels) the quotient below the clamp is < 2^22, so a float estimate
// N * rcp(D) is within 1 of N / D (four roundings of 2^-24 each) and one
// integer fix-up each way makes it the exact floor: a short dependency chain
// instead of a double division.  Larger q_max: the exact double quotient.
__device__ __forceinline__ unsigned regulate32(const Ctx &x, unsigned len, unsigned np, unsigned nt) {
  const unsigned long long N = (unsigned long long)len * nt * (unsigned long long)x.numA;
  const unsigned long long D = (unsigned long long)x.den * np;
  const unsigned qmax = (unsigned)x.qmax, qmin = (unsigned)x.qmin;
  if (x.qmax < (1LL << 22)) {
    if ((unsigned long long)(qmax + 1) * D <= N) return qmax;
    unsigned q = (unsigned)__fmul_rn(__ull2float_rn(N), __frcp_rn(__ull2float_rn(D)));
    q = q > qmax + 1 ? qmax + 1 : q;
    if ((unsigned long long)q * D > N) --q;
    else if ((unsigned long long)(q + 1) * D <= N) ++q;
    return q < qmin ? qmin : (q > qmax ? qmax : q);
  }
  if (N < (1ull << 53)) {
    // exact in one double division: N and D convert exactly, and for a
    // non-integer N/D the distance to the next integer (>= 1/D) exceeds the
    // rounding error (<= (N/D) 2^-53) because N < 2^53, so the floor is exact
    const double qd = floor(__ddiv_rn((double)N, (double)D));
    const double qc = fmin(fmax(qd, (double)x.qmin), (double)x.qmax);
    return (unsigned)qc;
  }
  if ((unsigned long long)(x.qmax + 1) * D <= N) return (unsigned)x.qmax;   // clamps high anyway
  long long q = (long long)__fdividef((float)N, (float)D);
  q = q < 0 ? 0 : (q > x.qmax + 1 ? x.qmax + 1 : q);
  while ((unsigned long long)q * D > N) --q;
  while ((unsigned long long)(q + 1) * D <= N) ++q;
  return (unsigned)(q < x.qmin ? x.qmin : (q > x.qmax ? x.qmax : q));
}

// regulate32 without 64-bit arithmetic (x.reg32x: numA, den < 2^24, q_max <
// 2^22, den * q_max < 2^29; the window invariants keep len, np, nt <= q_max + 1).
// The float quotient carries at most 7 roundings of 2^-24 (two products in
// the numerator, one in the denominator, __fdividef's 2 ulp), so below 2^22
// it is within 1.75 of N / D and its truncation within 2 of the exact floor:
// the remainder r = N - qe * D then lies in (-2D, 3D), fits 32 bits, and is
// computed from the low words alone; two compares each way make qe the exact
// floor.  An estimate far above the clamp returns q_max before the remainder
// (which would wrap) is looked at.
struct RegF {
  float numA, den, hi;
  unsigned numA32, den32, qmin, qmax;
};
__device__ __forceinline__ RegF make_regf(const Ctx &x) {
  RegF f;
  f.numA = (float)x.numA;
  f.den = (float)x.den;
  f.hi = (float)(x.qmax + 8);
  f.numA32 = (unsigned)x.numA;
  f.den32 = (unsigned)x.den;
  f.qmin = (unsigned)x.qmin;
  f.qmax = (unsigned)x.qmax;
  return f;
}
__device__ __forceinline__ unsigned regulate32x(const RegF &f, unsigned len, unsigned np, unsigned nt) {
  const float fn = __fmul_rn(__fmul_rn((float)len, (float)nt), f.numA);
  const float fd = __fmul_rn((float)np, f.den);
  const float qf = __fdividef(fn, fd);
  const unsigned qe = (unsigned)qf;   // truncation (saturating)
  const unsigned Nl = len * nt * f.numA32, Dl = np * f.den32;
  const int r = (int)(Nl - qe * Dl), D = (int)Dl;
  const int adj = (r >= D ? 1 : 0) + (r >= 2 * D ? 1 : 0) - (r < 0 ? 1 : 0) - (r < -D ? 1 : 0);
  unsigned q = qe + (unsigned)adj;
  q = qf > f.hi ? f.qmax : q;
  return min(max(q, f.qmin), f.qmax);
}

// regulate() through the 32-bit form whenever the operands fit (always for
// sensors up to 4.19M pixels): no double division on the candidate paths
__device__ __forceinline__ long long regulate_fast(const Ctx &x, long long len, long long np, long long nt) {
  if (len < (1LL << 32) && np < (1LL << 32) && nt < (1LL << 32)) {
    // (a window of at most q_max + 1 entries with nt <= np <= len -- every candidate window,
    // prediction and speculative start: no 64-bit arithmetic)
    if (x.reg32x && len <= x.qmax + 1 && np <= len && nt <= np && np >= 1)
      return (long long)regulate32x(make_regf(x), (unsigned)len, (unsigned)np, (unsigned)nt);
    return (long long)regulate32(x, (unsigned)len, (unsigned)np, (unsigned)nt);
  }
  return regulate(x, len, np, nt);
}

// parity surface for the regulator: regulate32x beside the exact 64-bit floor
// for arbitrary (len, np, nt) -- fibar_debug_regulate
__global__ void __launch_bounds__(TPB) k_debug_regulate(Ctx x, const unsigned *len, const unsigned *np, const unsigned *nt,
                                                        long long n, unsigned *out_fast, unsigned *out_exact) {
  const RegF rf = make_regf(x);
  for (long long i = (long long)blockIdx.x * TPB + threadIdx.x; i < n; i += (long long)gridDim.x * TPB) {
    out_fast[i] = regulate32x(rf, len[i], np[i], nt[i]);
    // the reference's integer formula (_kernels.py:195-201) in exact 64-bit arithmetic
    const unsigned long long N = (unsigned long long)len[i] * nt[i] * (unsigned long long)x.numA;
    const unsigned long long D = (unsigned long long)x.den * np[i];
    const unsigned long long q = N / D;
    out_exact[i] = (unsigned)(q < (unsigned long long)x.qmin ? (unsigned long long)x.qmin
                                                             : (q > (unsigned long long)x.qmax ? (unsigned long long)x.qmax : q));
  }
}

// The reference's per-event queue bookkeeping (_kernels.py:132-205) restated on
// the suffix window [s, j]: the push of event j activates its pixel / tile iff
// its previous same-pixel / same-tile event lies before s; the trim pops
// [s, j+1-q) and each popped k deactivates iff its next occurrence lies after j.
// k_window_run steps it per chunk lane, the verifier's re-runs per warp.

// Exact distinct-pixel / distinct-tile counts for every chunk's candidate
// windows [max(s_start, a_c - L_i), a_c - 1], as deltas from the previous
// chunk's window of the same candidate (one warp per chunk).
__global__ void __launch_bounds__(TPB) k_anchor(Ctx x) {
  pdl_wait();
  // counted against the predicted start state (bs->p_*); chunks 1..T, T being
  // the batch end (the next batch's prediction)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    x.bsn->p_geo = 0;              // set by k_anchor2 if a fixed point is unsettled
    x.bs->s_anchor = x.bs->p_s;    // (the window run reads this copy: p_s is rewritten three batches on)
  }
  const long long B = x.bs->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  const int lane = threadIdx.x & 31;
  const int c = (int)((blockIdx.x * (long long)TPB + threadIdx.x) >> 5) + 1;
  if (c > T) return;
  const long long E0 = x.bs->E0, s0 = x.bs->p_s, q0 = x.bs->p_q;
  const int nc = x.bs->p_geo ? NCAND : NLIN;   // geometric candidates only after an unsettled batch
  const long long a = anchor_at(x, E0, B, c, T);
  const long long Jc = a - 1;
  const long long ap = c == 1 ? E0 : anchor_at(x, E0, B, c - 1, T);
  const long long Jp = ap - 1;
  int cp[NCAND], ct[NCAND];
  int c0p = 0, c0t = 0;   // the no-pop window [s0, Jc] (a growing window: no eviction yet in the batch)
  long long sp[NCAND];
#pragma unroll
  for (int i = 0; i < NCAND; ++i) {
    cp[i] = 0;
    ct[i] = 0;
    sp[i] = c == 1 ? s0 : max(s0, ap - cand_len(x, q0, i));
  }
  // grow the right edge (Jp, Jc] with the previous starts
  for (long long k = Jp + 1 + lane; k <= Jc; k += 32) {
    const uint2 d = x.dp[k - E0];
    const unsigned long long k0 = (unsigned long long)(k - s0);
    c0p += (unsigned long long)d.x > k0;
    c0t += (unsigned long long)d.y > k0;
#pragma unroll
    for (int i = 0; i < NCAND; ++i) {
      if (i >= nc) break;
      const unsigned long long ks = (unsigned long long)(k - sp[i]);
      cp[i] += (unsigned long long)d.x > ks;
      ct[i] += (unsigned long long)d.y > ks;
    }
  }
  // shrink the left edge to the new starts (chunk 1's edges start at the batch's
  // whole start window and can be long: k_anchor_base counts those grid-wide)
#pragma unroll
  for (int i = 0; i < NCAND; ++i) {
    if (c == 1 || i >= nc) break;
    const long long sn = max(s0, a - cand_len(x, q0, i));
    for (long long k = sp[i] + lane; k < sn; k += 32) {
      const uint2 r = x.rnext[(unsigned long long)k & x.Rm];
      const unsigned long long dd = (unsigned long long)(Jc - k);
      cp[i] -= (unsigned long long)r.x > dd;
      ct[i] -= (unsigned long long)r.y > dd;
    }
  }
#pragma unroll
  for (int i = 0; i < NCAND; ++i) {
    if (i >= nc) break;
    const int vp = __reduce_add_sync(0xffffffffu, cp[i]);
    const int vt = __reduce_add_sync(0xffffffffu, ct[i]);
    if (lane == 0) x.anc[(long long)c * NCAND + i] = make_int2(vp, vt);
  }
  c0p = __reduce_add_sync(0xffffffffu, c0p);
  c0t = __reduce_add_sync(0xffffffffu, c0t);
  if (lane == 0) x.anc0[c] = make_int2(c0p, c0t);
}

// chunk 1's left edges [s_start, s_1i) counted by the whole grid (y = candidate)
__global__ void __launch_bounds__(TPB) k_anchor_base(Ctx x) {
  pdl_wait();
  __shared__ int red[2][TPB / 32];
  const long long B = x.bs->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  if (T < 1) return;
  const int i = blockIdx.y;
  if (i >= (x.bs->p_geo ? NCAND : NLIN)) return;
  const long long E0 = x.bs->E0, s0 = x.bs->p_s, q0 = x.bs->p_q;
  const long long a = anchor_at(x, E0, B, 1, T);
  const long long Jc = a - 1;
  const long long sn = max(s0, a - cand_len(x, q0, i));
  int cp = 0, ct = 0;
  for (long long k = s0 + (long long)blockIdx.x * TPB + threadIdx.x; k < sn; k += (long long)gridDim.x * TPB) {
    const uint2 r = x.rnext[(unsigned long long)k & x.Rm];
    const unsigned long long dd = (unsigned long long)(Jc - k);
    cp += (unsigned long long)r.x > dd;
    ct += (unsigned long long)r.y > dd;
  }
  cp = __reduce_add_sync(0xffffffffu, cp);
  ct = __reduce_add_sync(0xffffffffu, ct);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = cp;
    red[1][threadIdx.x >> 5] = ct;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int sp = 0, st = 0;
    for (int w = 0; w < TPB / 32; ++w) {
      sp += red[0][w];
      st += red[1][w];
    }
    if (sp) atomicSub(&x.anc[NCAND + i].x, sp);
    if (st) atomicSub(&x.anc[NCAND + i].y, st);
  }
}

// inclusive scan of the deltas over chunks, one CTA per candidate chain
// (chains interleaved with stride `nc` in `anc`)
__global__ void __launch_bounds__(1024) k_anchor_scan(Ctx x, int2 *anc, int nc) {
  pdl_wait();
  constexpr int PER = 4;
  __shared__ int2 wt[33];
  const long long B = x.bs->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  int i = blockIdx.x;
  if (anc == x.anc && i == NCAND) {   // the extra chain: the no-pop window counts
    anc = x.anc0;
    nc = 1;
    i = 0;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int2 carry = make_int2((int)x.bs->p_np, (int)x.bs->p_nt);
  for (int base = 1; base <= T; base += 1024 * PER) {
    const int c0 = base + threadIdx.x * PER;
    int2 v[PER];
    int2 tsum = make_int2(0, 0);
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      v[r] = c0 + r <= T ? anc[(long long)(c0 + r) * nc + i] : make_int2(0, 0);
      tsum.x += v[r].x;
      tsum.y += v[r].y;
    }
    int2 inc = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int tx = __shfl_up_sync(0xffffffffu, inc.x, o), ty = __shfl_up_sync(0xffffffffu, inc.y, o);
      if (lane >= o) {
        inc.x += tx;
        inc.y += ty;
      }
    }
    if (lane == 31) wt[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      const int2 w = wt[lane];
      int2 wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int tx = __shfl_up_sync(0xffffffffu, wi.x, o), ty = __shfl_up_sync(0xffffffffu, wi.y, o);
        if (lane >= o) {
          wi.x += tx;
          wi.y += ty;
        }
      }
      wt[lane] = make_int2(wi.x - w.x, wi.y - w.y);
      if (lane == 31) wt[32] = wi;
    }
    __syncthreads();
    int2 run = make_int2(carry.x + wt[wid].x + inc.x - tsum.x, carry.y + wt[wid].y + inc.y - tsum.y);
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      run.x += v[r].x;
      run.y += v[r].y;
      if (c0 + r <= T) anc[(long long)(c0 + r) * nc + i] = run;
    }
    carry.x += wt[32].x;
    carry.y += wt[32].y;
    __syncthreads();
  }
}

// Per chunk: locate the regulator's fixed point between the coarse candidate
// windows (largest stable candidate, G(L) >= L, and the next, unstable one) by
// linear interpolation of G(L) - L.  The fine candidates of pass 2 are centred
// on it.  In steady state the true window sits within a few dozen events of
// that fixed point and never far beyond it, so the first unstable fine
// candidate above the largest stable one is a start that collapses onto the
// true trajectory within a handful of events, with few evictions.
__device__ void fixed_point(const Ctx &x, int c, int T, long long &Lout, long long &uout, bool &unsettled) {
  const long long E0 = x.bs->E0, s0 = x.bs->p_s, q0 = x.bs->p_q;
  const long long a = anchor_at(x, E0, x.bs->B, c, T);
  unsettled = false;
  if (c == 0 || a == E0) {
    Lout = a - s0;
    uout = 32;
    return;
  }
  const int nc = x.bs->p_geo ? NCAND : NLIN;
  long long lens[NCAND], fs[NCAND];
#pragma unroll 1
  for (int i = 0; i < nc; ++i) {
    const long long len = a - max(s0, a - cand_len(x, q0, i));
    const int2 cnt = x.anc[(long long)c * NCAND + i];
    const long long f = (cnt.x >= 1 && cnt.y >= 1) ? regulate_fast(x, len, cnt.x, cnt.y) - len : -1;
    int k = i;   // insertion by length
    while (k > 0 && lens[k - 1] > len) {
      lens[k] = lens[k - 1];
      fs[k] = fs[k - 1];
      --k;
    }
    lens[k] = len;
    fs[k] = f;
  }
  long long len_lo = -1, len_hi = -1, f_lo = 0, f_hi = 0;
#pragma unroll 1
  for (int i = 0; i < nc; ++i) {
    if (fs[i] >= 0) {
      len_lo = lens[i];
      f_lo = fs[i];
      len_hi = -1;
    } else if (len_hi < 0 && lens[i] > len_lo) {
      len_hi = lens[i];
      f_hi = fs[i];
    }
  }
  long long L, unit = 32;
  if (len_lo < 0) {
    L = lens[0];                         // even the shortest candidate is unstable
  } else if (len_hi < 0) {
    L = len_lo;                          // longest candidate stable (e.g. growth from s_start)
  } else {
    const double root = (double)len_lo + (double)(len_hi - len_lo) * (double)f_lo / (double)(f_lo - f_hi);
    L = (long long)ceil(root);
    unit = max(32LL, (len_hi - len_lo) / 64);
  }
  // the next batch keeps the linear candidates only while every fixed point
  // stays well inside their span; a window still growing from the batch start
  // (clamped) is unsettled too: its target can run far from q0 next batch
  const bool clamped = len_lo >= 0 && len_hi < 0 && len_lo == a - s0;
  unsettled = clamped || L < q0 + c_lin_off[0] / 2 || L > q0 + c_lin_off[NLIN - 1] / 2;
  Lout = L;
  uout = unit;
}

// the fixed points of chunks 1..T, one thread each (large batches)
__global__ void __launch_bounds__(TPB) k_fp(Ctx x) {
  pdl_wait();
  const int T = (int)((x.bs->B + x.chunk - 1) / x.chunk);
  const int c = blockIdx.x * TPB + threadIdx.x + 1;
  if (c > T) return;
  long long L, u;
  bool uns;
  fixed_point(x, c, T, L, u, uns);
  x.lc[c] = L;
  x.lu[c] = u;
  if (uns) x.bsn->p_geo = 1;
}

__device__ __forceinline__ long long fine_start(const Ctx &x, long long s0, long long a, long long center,
                                                long long unit, int j) {
  long long L = center + c_fine_mul[j] * unit;
  L = L < 1 ? 1 : (L > x.qmax ? x.qmax : L);
  return max(s0, a - L);
}

// exact counts of every chunk's fine candidate windows [s_cj, a_c - 1], as
// deltas from the previous chunk's window of the same candidate (the start
// may move either way); one warp per chunk
__global__ void __launch_bounds__(TPB) k_anchor2(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  const int lane = threadIdx.x & 31;
  const int c = (int)((blockIdx.x * (long long)TPB + threadIdx.x) >> 5) + 1;
  if (c > T) return;   // chunks 1..T (T: the batch end, for the next batch's prediction)
  const long long E0 = x.bs->E0, s0 = x.bs->p_s;
  const long long ac = anchor_at(x, E0, B, c, T);
  const long long ap = c == 1 ? E0 : anchor_at(x, E0, B, c - 1, T);
  const long long Jc = ac - 1, Jp = ap - 1;
  // the regulator's fixed points of this chunk (lane 0) and the previous one
  // (lane 1), from the coarse counts; this chunk's goes to the window run
  long long fpL = 0, fpU = 32;
  bool uns = false;
  if (x.fp_fused) {   // small batches: no separate launch (k_fp computes them for large ones)
    if (lane < 2 && !(lane == 1 && c == 1)) fixed_point(x, c - lane, T, fpL, fpU, uns);
    if (lane == 0) {
      x.lc[c] = fpL;
      x.lu[c] = fpU;
      if (uns) x.bsn->p_geo = 1;
    }
  } else if (lane < 2 && !(lane == 1 && c == 1)) {
    fpL = x.lc[c - lane];
    fpU = x.lu[c - lane];
  }
  const long long lcc = __shfl_sync(0xffffffffu, fpL, 0), lcp = c == 1 ? 0 : __shfl_sync(0xffffffffu, fpL, 1);
  const long long luc = __shfl_sync(0xffffffffu, fpU, 0), lup = c == 1 ? 32 : __shfl_sync(0xffffffffu, fpU, 1);
  long long sp[NFINE];
  int cp[NFINE], ct[NFINE];
#pragma unroll
  for (int j = 0; j < NFINE; ++j) {
    sp[j] = c == 1 ? s0 : fine_start(x, s0, ap, lcp, lup, j);
    cp[j] = 0;
    ct[j] = 0;
  }
  for (long long k = Jp + 1 + lane; k <= Jc; k += 32) {
    const uint2 d = x.dp[k - E0];
#pragma unroll
    for (int j = 0; j < NFINE; ++j) {
      const unsigned long long ks = (unsigned long long)(k - sp[j]);
      cp[j] += (unsigned long long)d.x > ks;
      ct[j] += (unsigned long long)d.y > ks;
    }
  }
#pragma unroll
  for (int j = 0; j < NFINE; ++j) {
    const long long sn = fine_start(x, s0, ac, lcc, luc, j);
    const int sgn = sn >= sp[j] ? -1 : 1;
    const long long lo = min(sp[j], sn), hi = max(sp[j], sn);
    for (long long k = lo + lane; k < hi; k += 32) {
      const uint2 r = x.rnext[(unsigned long long)k & x.Rm];
      const unsigned long long dd = (unsigned long long)(Jc - k);
      cp[j] += sgn * (int)((unsigned long long)r.x > dd);
      ct[j] += sgn * (int)((unsigned long long)r.y > dd);
    }
  }
#pragma unroll
  for (int j = 0; j < NFINE; ++j) {
    const int vp = __reduce_add_sync(0xffffffffu, cp[j]);
    const int vt = __reduce_add_sync(0xffffffffu, ct[j]);
    if (lane == 0) x.anc2[(long long)c * NFINE + j] = make_int2(vp, vt);
  }
}

// The next batch's start prediction: the batch-end "chunk" T's start chosen
// exactly as k_window_run chooses a chunk start (the first unstable fine
// candidate above the largest stable one, or the no-pop window when stable),
// with its exact counts and regulated target.  One thread.
__global__ void k_predict(Ctx x) {
  pdl_wait();
  BatchState *b = x.bs, *n = x.bsn;
  const long long B = b->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  if (T == 0) {   // an empty batch: the same start
    n->p_s = b->p_s;
    n->p_q = b->p_q;
    n->p_np = b->p_np;
    n->p_nt = b->p_nt;
    n->p_geo = b->p_geo;
    return;
  }
  const long long s0 = b->p_s, a = b->E0 + B;
  const long long center = x.lc[T], unit = x.lu[T];
  int jstar = -1;
#pragma unroll 1
  for (int j = 0; j < NFINE; ++j) {
    const long long sc = fine_start(x, s0, a, center, unit, j);
    const int2 cnt = x.anc2[(long long)T * NFINE + j];
    const long long len = a - sc;
    if (cnt.x >= 1 && cnt.y >= 1 && regulate_fast(x, len, cnt.x, cnt.y) >= len) jstar = j;
  }
  const int g = jstar + 1 < NFINE ? jstar + 1 : NFINE - 1;
  int2 cnt = x.anc2[(long long)T * NFINE + g];
  long long ss = fine_start(x, s0, a, center, unit, g);
  const int2 c0 = x.anc0[T];
  const long long len0 = a - s0;
  if (c0.x >= 1 && c0.y >= 1 && regulate_fast(x, len0, c0.x, c0.y) >= len0) {
    ss = s0;
    cnt = c0;
  }
  const long long len = a - ss;
  n->p_s = ss;
  n->p_q = (cnt.x >= 1 && cnt.y >= 1) ? regulate_fast(x, len, cnt.x, cnt.y) : len;
  n->p_np = cnt.x;
  n->p_nt = cnt.y;
}

// One lane per chunk, the warp stepping its lanes' events in lockstep.  Each
// lane starts from the longest candidate window just past the regulator's
// fixed point (a too-long window collapses to the true one within a few
// events), warms up, then runs its own chunk.  Evictions of more than a few
// entries (the first trims of a long start window) are counted by the whole
// warp, 32 ring entries per step.

__global__ void __launch_bounds__(128) k_window_run(Ctx x) {
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) open_batch(x);   // the batch's true start (after the previous verifier)
  const long long B = x.bs->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  const int c = blockIdx.x * 128 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if ((blockIdx.x * 128 + (threadIdx.x & ~31)) >= T) return;   // whole warp out of range
  const bool valid = c < T;
  const DevState s = *x.st;
  const long long E0 = x.bs->E0;
  const long long s_true = s.s;             // chunk 0 starts exactly here
  const long long s_start0 = x.bs->s_anchor;   // the anchors' start: candidate windows are clamped to it
  const long long b = E0 + (long long)c * x.chunk;
  const long long e = valid ? min(E0 + B, b + x.chunk) : b;
  const long long a = valid ? chunk_warm_start(x, E0, c) : b;
  WState w{0, 1, 0, 0, 0};
  if (valid) {
    if (a == E0) {
      w.s = s_true;
      w.q = s.q;
      w.npix = s.npix;
      w.ntiles = s.ntiles;
      w.evctr = s.evctr;
    } else {
      const long long center = x.lc[c], unit = x.lu[c];
      int jstar = -1;
#pragma unroll 1
      for (int j = 0; j < NFINE; ++j) {
        const long long sc = fine_start(x, s_start0, a, center, unit, j);
        const int2 cnt = x.anc2[(long long)c * NFINE + j];
        const long long len = a - sc;
        if (cnt.x >= 1 && cnt.y >= 1 && regulate_fast(x, len, cnt.x, cnt.y) >= len) jstar = j;
      }
      const int g = jstar + 1 < NFINE ? jstar + 1 : NFINE - 1;
      int2 cnt = x.anc2[(long long)c * NFINE + g];
      w.s = fine_start(x, s_start0, a, center, unit, g);
      // a window still growing (no eviction yet in this batch: the cold start
      // or a rising target) has no fixed point near the candidates; its exact
      // state is the no-pop window [s_start, a - 1] whenever that is stable
      const int2 c0 = x.anc0[c];
      const long long len0 = a - s_start0;
      if (c0.x >= 1 && c0.y >= 1 && regulate_fast(x, len0, c0.x, c0.y) >= len0) {
        w.s = s_start0;
        cnt = c0;
      }
      w.npix = cnt.x;
      w.ntiles = cnt.y;
      const long long len = a - w.s;
      w.q = (cnt.x >= 1 && cnt.y >= 1) ? regulate_fast(x, len, cnt.x, cnt.y) : len;
      if (x.debug) {
        long long bn = 0, bt = 0;
        for (long long k = w.s; k < a; ++k) {
          const uint2 rr = x.rnext[(unsigned long long)k & x.Rm];
          bn += (unsigned long long)rr.x > (unsigned long long)(a - 1 - k);
          bt += (unsigned long long)rr.y > (unsigned long long)(a - 1 - k);
        }
        if (bn != w.npix || bt != w.ntiles) atomicAdd((unsigned long long *)&x.st->dbg_bad, 1ull);
      }
      w.evctr = (s.evctr + (a - E0)) % x.every;
    }
  }
  ChunkRec r;
  r.st_s = w.s;
  r.st_q = w.q;
  long long qlo = 0x7FFFFFFFFFFFFFFFLL, qhi = -1;
  long long wpops = 0, coop = 0;
  const unsigned n_my = (unsigned)(e - a);
  const unsigned n_max = __reduce_max_sync(0xffffffffu, n_my);
  // 32-bit state relative to the batch's start window (every index in play is
  // within B + window of it); ring slots as (slot of s_start + offset) & Rm.
  // S / Qt are stored relative to the true start (a lane whose trajectory is
  // still behind it is invalid and will be re-run by the verifier)
  const long long base = min(s_start0, s_true);
  const unsigned sofs = (unsigned)(s_true - base);
  const unsigned bslot = (unsigned)((unsigned long long)base & x.Rm);
  const unsigned rm = (unsigned)x.Rm;
  unsigned sr = (unsigned)(w.s - base);
  const unsigned ar = (unsigned)(a - base), br = (unsigned)(b - base);
  const unsigned e0r = (unsigned)(E0 - base);
  unsigned q = (unsigned)w.q;
  int np = (int)w.npix, nt = (int)w.ntiles;
  unsigned ev = (unsigned)w.evctr;
  const unsigned every = (unsigned)x.every;
  unsigned qlo32 = 0xFFFFFFFFu, qhi32 = 0;
  uint2 dnext = n_my > 0 ? x.dp[ar - e0r] : make_uint2(0, 0);
  for (unsigned t = 0; t < n_max; ++t) {
    const bool act = t < n_my;
    const unsigned jr = ar + t;
    if (act && jr == br) {
      r.st_s = base + sr;
      r.st_q = q;
    }
    unsigned lo = 0, hi = 0;
    if (act) {
      const uint2 d = dnext;
      if (t + 1 < n_my) dnext = x.dp[jr + 1 - e0r];
      const unsigned js = jr - sr;
      np += d.x > js;
      nt += d.y > js;
      if (js + 1 > q) {
        lo = sr;
        hi = jr + 1 - q;
      }
    }
    const bool big = hi - lo > 8;
    if (jr < br) wpops += hi - lo;
    if (!big && hi > lo) {
      // up to 8 entries, four independent loads in flight per round
      for (unsigned k = lo; k < hi; k += 4) {
        uint2 rr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) rr[u] = k + u < hi ? x.rnext[(bslot + k + u) & rm] : make_uint2(0u, 0u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned dd = jr - (k + u);
          np -= rr[u].x > dd;
          nt -= rr[u].y > dd;
        }
      }
      sr = hi;
    }
    // a long eviction (the collapse of a too-long speculative start): up to
    // WIN_SOLO entries each lane streams its own range with 8 loads in flight
    // (all lanes at once); longer ones are counted by the whole warp, 32
    // entries per step, one lane after another
    const bool huge = hi - lo > WIN_SOLO;
    unsigned m = __ballot_sync(0xffffffffu, huge);
    while (m) {
      const int L = __ffs(m) - 1;
      const unsigned l0 = __shfl_sync(0xffffffffu, lo, L);
      const unsigned h0 = __shfl_sync(0xffffffffu, hi, L);
      const unsigned jL = __shfl_sync(0xffffffffu, jr, L);
      int cp = 0, ct = 0;
      for (unsigned k = l0 + lane; k < h0; k += 32) {
        const uint2 rr = x.rnext[(bslot + k) & rm];
        const unsigned dd = jL - k;
        cp += rr.x > dd;
        ct += rr.y > dd;
      }
      cp = __reduce_add_sync(0xffffffffu, cp);
      ct = __reduce_add_sync(0xffffffffu, ct);
      ++coop;
      if (lane == L) {
        np -= cp;
        nt -= ct;
        sr = h0;
      }
      m &= m - 1;
    }
    if (big && !huge) {
      int cp = 0, ct = 0;
      for (unsigned k = lo; k < hi; k += 8) {
        uint2 rr[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) rr[u] = k + u < hi ? x.rnext[(bslot + k + u) & rm] : make_uint2(0u, 0u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (k + u >= hi) break;
          const unsigned dd = jr - (k + u);
          cp += rr[u].x > dd;
          ct += rr[u].y > dd;
        }
      }
      np -= cp;
      nt -= ct;
      sr = hi;
      ++coop;
    }
    if (act) {
      if (++ev >= every) {
        ev = 0;
        if (np >= 1 && nt >= 1) {
          q = regulate32(x, jr - sr + 1, (unsigned)np, (unsigned)nt);
          if (jr >= br) {
            qlo32 = min(qlo32, q);
            qhi32 = max(qhi32, q);
          }
        }
      }
      if (jr >= br) {
        x.S[jr - e0r] = sr - sofs;
        x.Qt[jr - e0r] = q;
      }
    }
  }
  w.s = base + sr;
  w.q = q;
  w.npix = np;
  w.ntiles = nt;
  w.evctr = ev;
  if (qhi32 > 0) {
    qlo = qlo32;
    qhi = qhi32;
  }
  {
    const unsigned long long wp = __reduce_add_sync(0xffffffffu, (unsigned)wpops);
    if (lane == 0) {
      atomicAdd((unsigned long long *)&x.st->warm_pops, wp);
      atomicAdd((unsigned long long *)&x.st->coop_iters, (unsigned long long)coop);
    }
  }
  if (!valid) return;
  r.en_s = w.s;
  r.en_q = w.q;
  r.en_np = w.npix;
  r.en_nt = w.ntiles;
  r.en_ev = w.evctr;
  r.qlo = qlo;
  r.qhi = qhi;
  x.ch[c] = r;
}

// The same run with G lanes per chunk (32 / G chunks per warp, still in
// lockstep).  The entries a window pops are always the next ones past its
// start, so the group keeps the G ring entries [s, s + G) in registers: lane u
// owns the positions = u (mod G) and holds the first one at or past s, loaded
// as soon as the previous one was popped (about G steps before the window start
// reaches it) -- the ring load leaves the step's dependency chain, an
// eviction of up to G entries is one compare per lane and a group reduction,
// and the fine candidates of the start state are evaluated G at a time.  Longer
// evictions (the collapse of a too-long start window) stream 8 entries per
// lane per round.  The warm-up and the chunk run as blocks of G steps: each
// lane loads one event's links per block (the steps take them by shuffle) and
// keeps one event's (S, Qt) to store.
template <int G>
__device__ __forceinline__ void window_run_g(const Ctx &x) {
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) open_batch(x);   // the batch's true start (after the previous verifier)
  constexpr int CPW = 32 / G;   // chunks per warp
  constexpr int V = 8;          // ring loads in flight per lane in a long eviction
  const long long B = x.bs->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  const int lane = threadIdx.x & 31, u = lane & (G - 1);
  const int cw = (blockIdx.x * 4 + (threadIdx.x >> 5)) * CPW;   // the warp's first chunk
  if (cw >= T) return;   // whole warp out of range
  const int c = cw + lane / G;
  const bool valid = c < T;
  const DevState s = *x.st;
  const long long E0 = x.bs->E0;
  const long long s_true = s.s;             // chunk 0 starts exactly here
  const long long s_start0 = x.bs->s_anchor;   // the anchors' start: candidate windows are clamped to it
  const long long b = E0 + (long long)c * x.chunk;
  const long long e = valid ? min(E0 + B, b + x.chunk) : b;
  const long long a = valid ? chunk_warm_start(x, E0, c) : b;
  const bool spec = valid && a != E0;
  WState w{0, 1, 0, 0, 0};
  // the speculative start: the fine candidates, G at a time
  int jstar = -1;
  long long center = 0, unit = 0;
  if (spec) {
    center = x.lc[c];
    unit = x.lu[c];
#pragma unroll 1
    for (int j = u; j < NFINE; j += G) {
      const long long sc = fine_start(x, s_start0, a, center, unit, j);
      const int2 cnt = x.anc2[(long long)c * NFINE + j];
      const long long len = a - sc;
      if (cnt.x >= 1 && cnt.y >= 1 && regulate_fast(x, len, cnt.x, cnt.y) >= len) jstar = j;
    }
  }
#pragma unroll
  for (int o = 1; o < G; o <<= 1) jstar = max(jstar, __shfl_xor_sync(0xffffffffu, jstar, o));
  if (valid) {
    if (!spec) {
      w.s = s_true;
      w.q = s.q;
      w.npix = s.npix;
      w.ntiles = s.ntiles;
      w.evctr = s.evctr;
    } else {
      const int g = jstar + 1 < NFINE ? jstar + 1 : NFINE - 1;
      int2 cnt = x.anc2[(long long)c * NFINE + g];
      w.s = fine_start(x, s_start0, a, center, unit, g);
      // a window still growing (no eviction yet in this batch) has no fixed
      // point near the candidates: the no-pop window [s_start, a - 1] whenever
      // that is stable (see k_window_run)
      const int2 c0 = x.anc0[c];
      const long long len0 = a - s_start0;
      if (c0.x >= 1 && c0.y >= 1 && regulate_fast(x, len0, c0.x, c0.y) >= len0) {
        w.s = s_start0;
        cnt = c0;
      }
      w.npix = cnt.x;
      w.ntiles = cnt.y;
      const long long len = a - w.s;
      w.q = (cnt.x >= 1 && cnt.y >= 1) ? regulate_fast(x, len, cnt.x, cnt.y) : len;
      if (x.debug && u == 0) {
        long long bn = 0, bt = 0;
        for (long long k = w.s; k < a; ++k) {
          const uint2 rr = x.rnext[(unsigned long long)k & x.Rm];
          bn += (unsigned long long)rr.x > (unsigned long long)(a - 1 - k);
          bt += (unsigned long long)rr.y > (unsigned long long)(a - 1 - k);
        }
        if (bn != w.npix || bt != w.ntiles) atomicAdd((unsigned long long *)&x.st->dbg_bad, 1ull);
      }
      w.evctr = (s.evctr + (a - E0)) % x.every;
    }
  }
  // 32-bit state relative to the batch's start window, as in k_window_run
  const long long base = min(s_start0, s_true);
  const unsigned sofs = (unsigned)(s_true - base);
  const unsigned bslot = (unsigned)((unsigned long long)base & x.Rm);
  const unsigned rm = (unsigned)x.Rm;
  unsigned sr = (unsigned)(w.s - base);
  const int ar = (int)(a - base), br = (int)(b - base), e0r = (int)(E0 - base);
  const int wl = br - ar, rl = (int)(e - b);   // this chunk's warm-up and run lengths
  unsigned q = (unsigned)w.q;
  int np = (int)w.npix, nt = (int)w.ntiles;
  unsigned ev = (unsigned)w.evctr;
  const unsigned every = (unsigned)x.every;
  const bool fastreg = x.reg32x != 0;
  const RegF rf = make_regf(x);
  unsigned qlo32 = 0xFFFFFFFFu, qhi32 = 0, coop = 0;
  const unsigned sr_first = sr;
  // this lane's ring entry: the first position = u (mod G) at or past sr,
  // reloaded as soon as it was popped (holding four entries per lane and
  // refilling between blocks measured slower: more instructions per step)
  unsigned pu = sr + (((unsigned)u - sr) & (unsigned)(G - 1));
  auto ring = [&](unsigned pos) { return x.rnext[(bslot + pos) & rm]; };
  uint2 e0 = ring(pu);
  const int gb = lane & ~(G - 1);   // the group's first lane

  // one event: push (d = its links), trim, re-target
  auto step = [&](bool act, int jr, unsigned dx, unsigned dy) -> bool {
    bool regd = false;
    unsigned hi = sr;
    const unsigned js = (unsigned)jr - sr;
    if (act) {
      np += dx > js;
      nt += dy > js;
      if (js + 1 > q) hi = (unsigned)jr + 1 - q;
    }
    // the eviction [sr, hi): this lane's held entries first
    unsigned cc = 0;   // pixels in the low half, tiles in the high half
    const unsigned pu0 = pu;
    if (pu < hi) {
      const uint2 en = e0;
      const unsigned dd = (unsigned)jr - pu;
      cc = (en.x > dd ? 1u : 0u) | (en.y > dd ? 0x10000u : 0u);
      pu += G;
    }
    // (butterfly: one redux.sync per group with sub-warp masks measured slower, run 43 -> 61 us)
#pragma unroll
    for (int o = 1; o < G; o <<= 1) cc += __shfl_xor_sync(0xffffffffu, cc, o);
    np -= (int)(cc & 0xFFFFu);
    nt -= (int)(cc >> 16);
    if (__ballot_sync(0xffffffffu, pu < hi)) {
      // more than G entries somewhere in the warp: V per lane per round
      int cp = 0, ct = 0;
      const unsigned n_u = pu < hi ? (hi - pu + G - 1) / G : 0u;
      for (unsigned i = 0; i < n_u; i += V) {
        uint2 rr[V];
#pragma unroll
        for (int v = 0; v < V; ++v)
          rr[v] = i + v < n_u ? x.rnext[(bslot + pu + (i + v) * G) & rm] : make_uint2(0u, 0u);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          if (i + v >= n_u) break;
          const unsigned dd = (unsigned)jr - (pu + (i + v) * G);
          cp += rr[v].x > dd;
          ct += rr[v].y > dd;
        }
      }
      pu += n_u * G;
#pragma unroll
      for (int o = 1; o < G; o <<= 1) {
        cp += __shfl_xor_sync(0xffffffffu, cp, o);
        ct += __shfl_xor_sync(0xffffffffu, ct, o);
      }
      np -= cp;
      nt -= ct;
      ++coop;
    }
    sr = hi;
    if (pu != pu0) e0 = ring(pu);   // needed once the window start passes it
    if (act) {
      if (++ev >= every) {
        ev = 0;
        if (np >= 1 && nt >= 1) {
          q = fastreg ? regulate32x(rf, (unsigned)jr - sr + 1, (unsigned)np, (unsigned)nt)
                      : regulate32(x, (unsigned)jr - sr + 1, (unsigned)np, (unsigned)nt);
          regd = true;
        }
      }
    }
    return regd;
  };

  // Warm-up, aligned so that every chunk of the warp ends it together: step t
  // of nw * G is event br - nw * G + t, active from the chunk's warm-up start.
  // Each lane loads the links of one event per block of G steps; the steps
  // take them by shuffle.
  const int wl_max = __reduce_max_sync(0xffffffffu, wl);
  const int nw = (wl_max + G - 1) / G;
#pragma unroll 1
  for (int t0 = 0; t0 < nw; ++t0) {
    const int j0 = br - (nw - t0) * G;
    const uint2 dv = j0 + u >= ar ? x.dp[j0 + u - e0r] : make_uint2(0u, 0u);
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const unsigned dx = __shfl_sync(0xffffffffu, dv.x, gb + k);
      const unsigned dy = __shfl_sync(0xffffffffu, dv.y, gb + k);
      step(j0 + k >= ar, j0 + k, dx, dy);
    }
  }
  ChunkRec r;
  r.st_s = base + sr;   // state after event b - 1: the chunk's speculative start
  r.st_q = q;
  const unsigned wpops = sr - sr_first;
  // The chunk itself: the window start and target after each event are kept
  // by the lane whose index the event has in its block, and stored per block.
  const int rl_max = __reduce_max_sync(0xffffffffu, rl);
  const int nr = (rl_max + G - 1) / G;
#pragma unroll 1
  for (int t0 = 0; t0 < nr; ++t0) {
    const int j0 = br + t0 * G;
    const bool mine = t0 * G + u < rl;
    const uint2 dv = mine ? x.dp[j0 + u - e0r] : make_uint2(0u, 0u);
    unsigned sv = 0, qv = 0;
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const unsigned dx = __shfl_sync(0xffffffffu, dv.x, gb + k);
      const unsigned dy = __shfl_sync(0xffffffffu, dv.y, gb + k);
      const bool act = t0 * G + k < rl;
      if (step(act, j0 + k, dx, dy)) {
        qlo32 = min(qlo32, q);
        qhi32 = max(qhi32, q);
      }
      if (k == u) {
        sv = sr - sofs;
        qv = q;
      }
    }
    if (mine) {
      x.S[j0 + u - e0r] = sv;
      x.Qt[j0 + u - e0r] = qv;
    }
  }
  {
    const unsigned wp = __reduce_add_sync(0xffffffffu, u == 0 ? wpops : 0u);
    const unsigned cp = __reduce_max_sync(0xffffffffu, coop);
    if (lane == 0) {
      atomicAdd((unsigned long long *)&x.st->warm_pops, (unsigned long long)wp);
      atomicAdd((unsigned long long *)&x.st->coop_iters, (unsigned long long)cp);
    }
  }
  if (!valid || u != 0) return;
  r.en_s = base + sr;
  r.en_q = q;
  r.en_np = np;
  r.en_nt = nt;
  r.en_ev = ev;
  r.qlo = qhi32 > 0 ? (long long)qlo32 : 0x7FFFFFFFFFFFFFFFLL;
  r.qhi = qhi32 > 0 ? (long long)qhi32 : -1;
  x.ch[c] = r;
}
__global__ void __launch_bounds__(128) k_window_run_g2(Ctx x) { window_run_g<2>(x); }
__global__ void __launch_bounds__(128) k_window_run_g4(Ctx x) { window_run_g<4>(x); }
__global__ void __launch_bounds__(128) k_window_run_g8(Ctx x) { window_run_g<8>(x); }

// Verify chunk boundaries: a chunk is exact once its speculative start state
// equals its predecessor's end state and the predecessor is exact.  Rounds
// re-run, in parallel, every chunk whose start disagrees with its
// predecessor's current end (read before the round writes anything), until
// every boundary agrees; each round makes at least the first disagreeing
// chunk exact, so this is exact by induction whatever the guesses.  Then the
// targets' extrema are reduced and the batch's final window state published.
//
// One thread-block cluster (VF_CTAS CTAs, hardware cluster barriers between
// the phases of a round): every boundary is checked by the whole cluster, and
// each re-run is done by one warp that stages the chunk's links dp[b, e) and
// the ring next-links of the evictions it will most likely make,
// [s, s + VF_RN), in shared memory with coalesced loads, after which lane 0
// steps the recurrence from shared memory.
constexpr int VF_DP = 64;     // >= the largest chunk
constexpr int VF_RN = 128;    // staged ring entries per re-run

// cluster-wide barrier; release / acquire at cluster scope also orders the
// CTAs' global-memory accesses
__device__ __forceinline__ void vf_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 32-bit state relative to the batch's start window (every index in play is
// within B + window of it), as in k_window_run.  The speculative run recorded
// (S, Qt) -- window start and target after each of the chunk's events; a
// re-run that reaches the same (s, q) after some event has merged with that
// trajectory (the distinct counts are functions of (s, j), the regulation
// counter of j), so the rest of the chunk and its end state stand as they are:
// the re-run stops there (regulation every event only).  Returns whether it
// merged.
// Returns 0: re-run, end changed; 1: merged with the recorded trajectory;
// 2: skipped (its start lies behind the batch's true start: an invalid
// trajectory's end, re-run once that predecessor is)
__device__ int rerun_chunk_staged(const Ctx &x, WState &w, long long b, long long e, long long E0, long long s_start,
                                  uint2 *sdp, uint2 *srn, uint2 *ssq, long long &qlo, long long &qhi) {
  const int lane = threadIdx.x & 31;
  if (w.s < s_start) return 2;
  const long long rn0 = w.s;
  for (int i = lane; i < (int)(e - b); i += 32) {
    sdp[i] = x.dp[b - E0 + i];
    ssq[i] = make_uint2(x.S[b - E0 + i], x.Qt[b - E0 + i]);
  }
  uint2 rr[VF_RN / 32];
#pragma unroll
  for (int u = 0; u < VF_RN / 32; ++u) rr[u] = x.rnext[(unsigned long long)(rn0 + lane + 32 * u) & x.Rm];
#pragma unroll
  for (int u = 0; u < VF_RN / 32; ++u) srn[lane + 32 * u] = rr[u];
  __syncwarp();
  unsigned merged_at = 0xFFFFFFFFu;
  if (lane == 0) {
    const unsigned bslot = (unsigned)((unsigned long long)s_start & x.Rm), rm = (unsigned)x.Rm;
    const unsigned r0 = (unsigned)(rn0 - s_start);   // first staged entry, relative
    const unsigned br = (unsigned)(b - s_start), er = (unsigned)(e - s_start), e0r = (unsigned)(E0 - s_start);
    const unsigned every = (unsigned)x.every;
    unsigned sr = (unsigned)(w.s - s_start), q = (unsigned)w.q, ev = (unsigned)w.evctr;
    int np = (int)w.npix, nt = (int)w.ntiles;
    unsigned qlo32 = 0xFFFFFFFFu, qhi32 = 0;
    const bool fastreg = x.reg32x != 0;
    const RegF rf = make_regf(x);
#pragma unroll 1
    for (unsigned jr = br; jr < er; ++jr) {
      const uint2 d = sdp[jr - br];
      const unsigned js = jr - sr;
      np += d.x > js;
      nt += d.y > js;
      if (js >= q) {   // the trim pops [sr, jr + 1 - q)
        const unsigned hi = jr + 1 - q;
#pragma unroll 1
        for (unsigned k = sr; k < hi; ++k) {
          const unsigned o = k - r0;
          const uint2 r = o < (unsigned)VF_RN ? srn[o] : x.rnext[(bslot + k) & rm];
          const unsigned dd = jr - k;
          np -= r.x > dd;
          nt -= r.y > dd;
        }
        sr = hi;
      }
      if (++ev >= every) {
        ev = 0;
        if (np >= 1 && nt >= 1) {
          q = fastreg ? regulate32x(rf, jr - sr + 1, (unsigned)np, (unsigned)nt)
                      : regulate32(x, jr - sr + 1, (unsigned)np, (unsigned)nt);
          qlo32 = min(qlo32, q);
          qhi32 = max(qhi32, q);
        }
      }
      const uint2 old = ssq[jr - br];
      if (every == 1 && old.x == sr && old.y == q) {
        merged_at = jr - br;
        break;
      }
      x.S[jr - e0r] = sr;
      x.Qt[jr - e0r] = q;
    }
    w.s = s_start + sr;
    w.q = q;
    w.npix = np;
    w.ntiles = nt;
    w.evctr = ev;
    if (qhi32 > 0) {
      qlo = qlo32;
      qhi = qhi32;
    }
  }
  merged_at = __shfl_sync(0xffffffffu, merged_at, 0);
  if (merged_at != 0xFFFFFFFFu) {
    // the chunk's targets after the merge are the recorded ones
    unsigned lo = 0xFFFFFFFFu, hi = 0;
    for (unsigned i = merged_at + 1 + lane; i < (unsigned)(e - b); i += 32) {
      lo = min(lo, ssq[i].y);
      hi = max(hi, ssq[i].y);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (hi > 0) {
      qlo = min(qlo, (long long)lo);
      qhi = max(qhi, (long long)hi);
    }
  }
  __syncwarp();
  return merged_at != 0xFFFFFFFFu ? 1 : 0;
}

__global__ void __launch_bounds__(VF_TPB, VF_TPB > 256 ? 1 : 2) k_window_verify(Ctx x) {
  pdl_wait();
  constexpr int NW = VF_TPB / 32;
  __shared__ uint2 sdp[NW][VF_DP];
  __shared__ uint2 ssq[NW][VF_DP];
  __shared__ uint2 srn[NW][VF_RN];
  __shared__ long long red_lo[NW], red_hi[NW];
  BatchState *bs = x.bs;
  const long long B = bs->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  const long long E0 = bs->E0, s_start = bs->s_start;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long tid = (long long)blockIdx.x * VF_TPB + threadIdx.x, nthr = (long long)gridDim.x * VF_TPB;
  const long long gw = (long long)blockIdx.x * NW + wid, nwarps = (long long)gridDim.x * NW;
  int rounds = 0;
  long long reruns = 0;
  // round 0 lists every disagreeing boundary; a re-run that did not merge
  // with its recorded trajectory changed its end state, so it lists its
  // successor for the next round itself (with that end state as the start)
  for (long long c = 1 + tid; c < T; c += nthr) {
    const ChunkRec &p = x.ch[c - 1];
    const ChunkRec &q = x.ch[c];
    if (q.st_s != p.en_s || q.st_q != p.en_q) {
      const unsigned i = atomicAdd(&bs->vcnt[0], 1u);
      VRec v;
      v.s = p.en_s;
      v.q = p.en_q;
      v.np = p.en_np;
      v.nt = p.en_nt;
      v.ev = p.en_ev;
      v.c = (int)c;
      v.pad = 0;
      x.vl[i] = v;
    }
  }
  vf_barrier();
  for (;; ++rounds) {
    const unsigned n = ld_relaxed_u32(&bs->vcnt[rounds % 3]);
    if (n == 0) break;
    reruns += n;
    if (tid == 0) bs->vcnt[(rounds + 2) % 3] = 0;   // for round r + 2 (its last reader passed a barrier)
    const VRec *in = x.vl + (long long)(rounds & 1) * T;
    VRec *out = x.vl + (long long)((rounds + 1) & 1) * T;
    unsigned *out_cnt = &bs->vcnt[(rounds + 1) % 3];
    for (long long i = gw; i < n; i += nwarps) {
      const VRec v = in[i];
      WState w{v.s, v.q, v.np, v.nt, v.ev};
      long long qlo = 0x7FFFFFFFFFFFFFFFLL, qhi = -1;
      const long long b = E0 + (long long)v.c * x.chunk;
      const long long e = min(E0 + B, b + x.chunk);
      const int how = rerun_chunk_staged(x, w, b, e, E0, s_start, sdp[wid], srn[wid], ssq[wid], qlo, qhi);
      const bool merged = how == 1;
      if (lane == 0 && how != 2) {
        ChunkRec r = x.ch[v.c];   // merged: the recorded end state stands
        r.st_s = v.s;
        r.st_q = v.q;
        if (!merged) {
          r.en_s = w.s;
          r.en_q = w.q;
          r.en_np = w.npix;
          r.en_nt = w.ntiles;
          r.en_ev = w.evctr;
          if (v.c + 1 < T) {
            VRec nx;
            nx.s = w.s;
            nx.q = w.q;
            nx.np = w.npix;
            nx.nt = w.ntiles;
            nx.ev = w.evctr;
            nx.c = v.c + 1;
            nx.pad = 0;
            out[atomicAdd(out_cnt, 1u)] = nx;
          }
        }
        r.qlo = qlo;
        r.qhi = qhi;
        x.ch[v.c] = r;
      }
    }
    vf_barrier();
  }
  // the targets' extrema over every chunk
  long long lo = 0x7FFFFFFFFFFFFFFFLL, hi = -1;
  for (long long c = tid; c < T; c += nthr) {
    lo = min(lo, x.ch[c].qlo);
    hi = max(hi, x.ch[c].qhi);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane == 0) {
    red_lo[wid] = lo;
    red_hi[wid] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < NW; ++w) {
      lo = min(lo, red_lo[w]);
      hi = max(hi, red_hi[w]);
    }
    if (hi >= 0) {
      atomicMin((unsigned long long *)&bs->qlo, (unsigned long long)lo);
      atomicMax((long long *)&bs->qhi, hi);
    }
  }
  vf_barrier();
  if (tid == 0) {
    DevState *s = x.st;
    if (T > 0) {
      const ChunkRec &r = x.ch[T - 1];
      s->s = r.en_s;
      s->q = r.en_q;
      s->npix = r.en_np;
      s->ntiles = r.en_nt;
      s->evctr = r.en_ev;
      if (bs->qhi >= 0) {
        s->qtmin = min(s->qtmin, bs->qlo);
        s->qtmax = max(s->qtmax, bs->qhi);
      }
      s->pops += r.en_s - s_start;
      bs->npop = r.en_s - s_start;
    } else {
      bs->npop = 0;
    }
    s->chunks += T;
    s->fix_rounds += rounds;
    s->mismatch += reruns;

  }
}

// ----------------------------------------------------------------- stale ---

// Every window entry popped in this batch becomes an item, in pop order (the
// order the reference blurs them, _kernels.py:152-189).  An entry is stale iff
// its pixel has no later event up to the popping event.
// Event jj pops the evictions [S[jj-1], S[jj]) (S is the window start after
// each event): one thread per event writes jj for its range, ranges longer
// than a warp (a collapsing window) written by the whole warp.  Replaces a
// binary search of S per eviction.
__global__ void __launch_bounds__(TPB) k_popj_map(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const unsigned jj = blockIdx.x * TPB + threadIdx.x;
  const int lane = threadIdx.x & 31;
  unsigned lo = 0, hi = 0;
  if (jj < B) {
    lo = jj == 0 ? 0u : x.S[jj - 1];
    hi = x.S[jj];
  }
  if (hi - lo <= 32)
    for (unsigned p = lo; p < hi; ++p) x.pmap[p] = jj;
  unsigned m = __ballot_sync(0xffffffffu, hi - lo > 32);
  while (m) {
    const int L = __ffs(m) - 1;
    const unsigned l0 = __shfl_sync(0xffffffffu, lo, L), h0 = __shfl_sync(0xffffffffu, hi, L);
    const unsigned j0 = __shfl_sync(0xffffffffu, jj, L);
    for (unsigned p = l0 + lane; p < h0; p += 32) x.pmap[p] = j0;
    m &= m - 1;
  }
}

__global__ void __launch_bounds__(TPB) k_popj(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const long long E0 = x.bs->E0, s_start = x.bs->s_start;
  const unsigned npop = B > 0 ? x.S[B - 1] : 0u;
  // one thread per eviction (balanced); the grid is sized for the batch's
  // events (about one eviction each) and strides over a collapsing window's
  unsigned nst = 0;
  for (unsigned p = blockIdx.x * TPB + threadIdx.x; p < npop; p += gridDim.x * TPB) {
    const unsigned lo = x.pmap[p];   // popping event (k_popj_map)
    const long long k = s_start + p;
    const long long j = E0 + lo;
    const bool stale = (unsigned long long)x.rnext[(unsigned long long)k & x.Rm].x > (unsigned long long)(j - k);
    const unsigned c = x.rkey[(unsigned long long)k & x.Rm];
    atomicSub(&x.wcnt[c], 1u);   // the entry leaves the window (H7 bookkeeping)
    Item it;
    it.jrel = lo;
    it.pix = FIBAR_NONE;
    it.runpos = FIBAR_NONE;
    it.pad = 0;
    if (stale) {
      it.pix = c;
      if (k < E0) {
        x.pt[c].carried = p;
        // no event of the pixel in this batch after its pre-batch last one
        if ((unsigned long long)x.rnext[(unsigned long long)k & x.Rm].x > (unsigned long long)(E0 + B - 1 - k)) {
          it.pad |= ITEM_CARRIED_ONLY;
          x.colist[atomicAdd(&x.bs->nco, 1u)] = p;   // resolved by k_blur_prep from this list
        }
      }
      ++nst;
    } else {
      x.prep[p].okm = 0;   // not blurred: the blur lanes skip it
    }
    x.item[p] = it;
  }
  nst = __reduce_add_sync(0xffffffffu, nst);
  if ((threadIdx.x & 31) == 0 && nst) atomicAdd((unsigned long long *)&x.bs->stale_batch, (unsigned long long)nst);
}


}  // namespace fibar
