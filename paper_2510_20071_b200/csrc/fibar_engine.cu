// fibar_engine.cu -- B200-native FIBAR reconstruction engine (sm_100a) + C ABI.
//
// One device batch (coalesced packets) flows through:
//   ingest     k_count_inb / k_compact      OOB filter + compaction (pipeline.py:516-528),
//                                            pixel keys, ring of window keys
//   group      radix_sort_pairs              stable (tile-major key, index) sort
//   link       k_seg_marks / k_link          per event: distance to previous same-pixel /
//                                            same-tile event; per ring slot: distance to next
//   window     k_anchor / k_anchor_scan /    the reference's FIFO window (_kernels.py:132-205)
//              k_fp / k_anchor2 /            reproduced exactly by chunked speculation +
//              k_window_run / k_window_fix   verification
//   stale      k_popj                        eviction event of every popped entry; stale iff
//                                            the pixel has no later event before its eviction
//   temporal   k_posinfo / k_temporal_runs / per-pixel in-order replay of the two-stage IIR
//              k_temporal_long               (_kernels.py:62-73 / 120-130), bit exact;
//                                            last-touch tables for the next batch
//   blur       k_blur_prep / k_blur          3x3 renormalised blur of stale pixels in eviction
//                                            order (_kernels.py:173-189), dataflow over a
//                                            persistent grid polling (epoch | value) words
//   final      k_final / k_batch_end         end-of-batch brightness, counters
//   read-out   k_sel_init / k_sel_hist /     exact percentile select + float64 map
//              k_render_map                  (pipeline.py:562-584)
//
// Filter ON, the blur stage of batch k runs on a second stream while batch k+1's
// front end runs; small batches replay a captured CUDA graph
// (4.6); consecutive kernels use programmatic dependent launch (pdl_wait()).
// Float32 arithmetic uses __fmul_rn/__fadd_rn (never contracted to FMA) so the
// result is bit-identical to the reference's strict-IEEE numba kernels.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <algorithm>
#include <string>
#include <vector>

#include "fibar_common.cuh"
#include "fibar_internal.h"
#include "../../include/fibar_b200.h"

using namespace fibar;

namespace fibar {
thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char *where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return FIBAR_E_CUDA;
}
}  // namespace fibar

namespace {

constexpr int NFINE = 10;     // fine candidate windows around the interpolated fixed point
constexpr int CHUNK_MIN = 32;  // smallest speculative window chunk (sizes the chunk arrays)
constexpr int NLIN = 7;      // coarse candidates q0 + c_lin_off[i]
constexpr int NGEO = 12;     // coarse candidates q0 * c_geo_mul[i]
constexpr int NCAND = NLIN + NGEO;
constexpr int TPB = 256;
constexpr unsigned ITEM_CARRIED_ONLY = 1u;   // Item.pad flag


__constant__ long long c_fine_mul[NFINE] = {-8, -4, -2, -1, 0, 1, 2, 4, 8, 16};
__constant__ long long c_lin_off[NLIN] = {-16384, -4096, -1024, 0, 1024, 4096, 16384};
__constant__ double c_geo_mul[NGEO] = {0.25, 0.5, 0.75, 1.25, 1.5, 2.0, 2.5, 3.0, 4.0, 6.0, 8.0, 12.0};

struct ChunkRec {
  long long st_s, st_q;                          // state after event b_c - 1 (speculative start)
  long long en_s, en_q, en_np, en_nt, en_ev;     // state after the chunk's last event
  long long qlo, qhi;                            // extrema of the targets set inside the chunk
};

struct SelState {
  unsigned prefix[4];
  unsigned rank[4];
  unsigned hist[4][2048];
  double lo, hi;
  int degenerate;
  unsigned done;   // blocks finished with the current histogram pass
};

struct Ctx {
  int W, H, ts, tiles_x, A;
  unsigned band_y0, full_H;   // row band [band_y0, band_y0 + H) of a full_H-row sensor
  long long n_pix;
  long long num, den, qmin, qmax, every;
  long long numA;   // num * A (tile area)
  float alpha, oma, beta, h;
  int use_gain, blur_on, spatial;
  DevState *st;
  BatchState *bs;     // this batch's scalars (parity buffer)
  long long *plast;   // per pixel: last event index before the batch
  unsigned *wcnt;     // per pixel: exact in-window event count (saturation check)
  float *pbar, *l;
  const float *gain;
  PixRec *pt;
  long long *last_tile;
  uint2 *ptt;
  unsigned *rkey;
  uint2 *rnext;
  unsigned long long Rm;
  const uint16_t *raw_x, *raw_y;
  const int8_t *raw_p;
  long long n_raw;
  unsigned *blockcnt;
  unsigned *ekey;
  int8_t *epol, *spol;
  uint2 *longseg;
  unsigned *tkey;                 // unsorted tile-major keys (sort input)
  const unsigned *skey, *sidx;    // sorted keys / batch-local event index
  uint2 *dp;
  unsigned *S;
  Item *item;
  PosRec *posrec;
  float *t2;
  unsigned long long *bv64, *mv64;   // (epoch << 32 | float bits) per blur item / per sorted position
  BlurPrep *prep;
  int chunk, warm, debug;
  int twarm;                  // warm-up events of a speculative long-segment piece
  unsigned blur_sleep;
  unsigned long long *dbg_t, *dbg_g;
  int2 *anc, *anc2;
  long long *lc, *lu;
  ChunkRec *ch;
};

// ---------------------------------------------------------------- ingest ---

constexpr int IN_ITEMS = 8;
constexpr int IN_TILE = TPB * IN_ITEMS;

// an event is kept iff it lies on the sensor (else it is out of bounds,
// counted like pipeline.py:524-525) and in this engine's row band (a band
// engine silently leaves other bands' events to their owners)
__device__ __forceinline__ bool on_sensor(const Ctx &x, unsigned xx, unsigned yy) {
  return xx < (unsigned)x.W && yy < x.full_H;
}
__device__ __forceinline__ bool in_band(const Ctx &x, unsigned yy) { return yy - x.band_y0 < (unsigned)x.H; }

__global__ void __launch_bounds__(TPB) k_count_inb(Ctx x, int nblocks) {
  pdl_wait();
  __shared__ unsigned wsum[TPB / 32], woob[TPB / 32];
  const long long base = (long long)blockIdx.x * IN_TILE + threadIdx.x * IN_ITEMS;
  unsigned cnt = 0, oob = 0;
#pragma unroll
  for (int r = 0; r < IN_ITEMS; ++r) {
    long long i = base + r;
    if (i < x.n_raw) {
      const unsigned xx = x.raw_x[i], yy = x.raw_y[i];
      const bool ok = on_sensor(x, xx, yy);
      oob += !ok;
      cnt += ok && in_band(x, yy);
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

__global__ void __launch_bounds__(TPB) k_compact(Ctx x, int nblocks) {
  pdl_wait();
  __shared__ unsigned wsum[TPB / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long E0 = x.st->E;
  const long long base = (long long)blockIdx.x * IN_TILE + threadIdx.x * IN_ITEMS;
  bool keep[IN_ITEMS];
  unsigned cnt = 0;
#pragma unroll
  for (int r = 0; r < IN_ITEMS; ++r) {
    long long i = base + r;
    keep[r] = i < x.n_raw && on_sensor(x, x.raw_x[i], x.raw_y[i]) && in_band(x, x.raw_y[i]);
    cnt += keep[r];
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
  unsigned pos = x.blockcnt[blockIdx.x] + wofs + incl - cnt;
#pragma unroll
  for (int r = 0; r < IN_ITEMS; ++r) {
    if (!keep[r]) continue;
    long long i = base + r;
    const unsigned xx = x.raw_x[i], yy = x.raw_y[i] - x.band_y0;
    const unsigned key = yy * (unsigned)x.W + xx;
    const unsigned tile = (yy / x.ts) * (unsigned)x.tiles_x + xx / x.ts;
    const unsigned sub = (yy % x.ts) * x.ts + xx % x.ts;
    x.ekey[pos] = key;
    x.tkey[pos] = tile * (unsigned)x.A + sub;
    x.epol[pos] = x.raw_p[i];
    if (x.spatial) x.rkey[(unsigned long long)(E0 + pos) & x.Rm] = key;
    ++pos;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    DevState *s = x.st;
    BatchState *b = x.bs;
    b->E0 = s->E;
    b->B = x.blockcnt[nblocks];
    b->s_start = s->s;
    b->npop = 0;
    b->stale_batch = 0;
    b->ticket = 0;
    b->nlong = 0;
    s->epoch += 1;
    b->epoch = s->epoch;
  }
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
  if (tr.y - tr.x <= 64) {
    unsigned best_lo = 0, best_hi = 0xFFFFFFFFu;
    bool have_lo = false;
    for (unsigned q = tr.x; q < tr.y; ++q) {
      unsigned o = x.sidx[q];
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
  if (first_tile) prev_t = x.last_tile[t];

  x.dp[jj] = make_uint2(dist32(j, prev_p), dist32(j, prev_t));
  x.rnext[(unsigned long long)j & x.Rm] =
      make_uint2(next_p < 0 ? FIBAR_INF32 : (unsigned)(next_p - j), next_t < 0 ? FIBAR_INF32 : (unsigned)(next_t - j));
  if (first_pix) {
    // the reference's active_count saturates at 65535, after which
    // its count-based staleness departs from this exact restatement.  wcnt is
    // the pixel's exact in-window event count at batch start; the count seen
    // by its t-th event this batch is at most wcnt + t, so a batch can only
    // reach the cap if wcnt + seglen > 65535 -- flag that (never misses).
    const unsigned seglen = x.pt[c].end - (unsigned)i;
    const unsigned wc = x.wcnt[c];
    if ((unsigned long long)wc + seglen > 65535ull) atomicAdd((unsigned long long *)&x.st->saturated, 1ull);
    x.wcnt[c] = wc + seglen;
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

// coarse candidate i: a dense linear grid around the batch-start target q0
// plus a geometric one that reaches windows far from it (cold start, scene change)
__device__ __forceinline__ long long cand_len(const Ctx &x, long long q0, int i) {
  long long L = i < NLIN ? q0 + c_lin_off[i] : (long long)((double)q0 * c_geo_mul[i - NLIN]);
  return L < 1 ? 1 : (L > x.qmax ? x.qmax : L);
}

// floor(N / D) for N >= 0, D > 0: a float32 reciprocal estimate (relative
// error ~1e-7, and the quotients here stay below 2^24) and an exact integer fix-up
__device__ __forceinline__ long long floordiv_nn(long long N, long long D) {
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
// multiply, num * A folded on the host, an approximate float quotient (a few
// units off at most below 2^24) fixed up exactly in integers
__device__ __forceinline__ unsigned regulate32(const Ctx &x, unsigned len, unsigned np, unsigned nt) {
  const unsigned long long N = (unsigned long long)len * nt * (unsigned long long)x.numA;
  const unsigned long long D = (unsigned long long)x.den * np;
  if ((unsigned long long)(x.qmax + 1) * D <= N) return (unsigned)x.qmax;   // clamps high anyway
  long long q = (long long)__fdividef((float)N, (float)D);
  q = q < 0 ? 0 : (q > x.qmax + 1 ? x.qmax + 1 : q);
  while ((unsigned long long)q * D > N) --q;
  while ((unsigned long long)(q + 1) * D <= N) ++q;
  return (unsigned)(q < x.qmin ? x.qmin : (q > x.qmax ? x.qmax : q));
}

// The reference's per-event queue bookkeeping (_kernels.py:132-205) restated on
// the suffix window [s, j]: the push of event j activates its pixel / tile iff
// its previous same-pixel / same-tile event lies before s; the trim pops
// [s, j+1-q) and each popped k deactivates iff its next occurrence lies after j.
// Scalar form, used by the verifier's re-runs.
__device__ void run_window(const Ctx &x, WState &w, long long jf, long long jt, long long E0, long long s_start,
                           bool write, long long &qlo, long long &qhi) {
  for (long long j = jf; j < jt; ++j) {
    const uint2 d = x.dp[j - E0];
    const unsigned long long js = (unsigned long long)(j - w.s);
    w.npix += (unsigned long long)d.x > js;
    w.ntiles += (unsigned long long)d.y > js;
    long long len = j - w.s + 1;
    if (len > w.q) {
      const long long snew = j + 1 - w.q;
      long long np = w.npix, nt = w.ntiles;
      for (long long k = w.s; k < snew; ++k) {
        const uint2 r = x.rnext[(unsigned long long)k & x.Rm];
        const unsigned long long dd = (unsigned long long)(j - k);
        np -= (unsigned long long)r.x > dd;
        nt -= (unsigned long long)r.y > dd;
      }
      w.npix = np;
      w.ntiles = nt;
      w.s = snew;
      len = w.q;
    }
    if (++w.evctr >= x.every) {
      w.evctr = 0;
      if (w.npix >= 1 && w.ntiles >= 1) {
        const long long qn = regulate(x, len, w.npix, w.ntiles);
        w.q = qn;
        qlo = min(qlo, qn);
        qhi = max(qhi, qn);
      }
    }
    if (write) x.S[j - E0] = (unsigned)(w.s - s_start);
  }
}

// Exact distinct-pixel / distinct-tile counts for every chunk's candidate
// windows [max(s_start, a_c - L_i), a_c - 1], as deltas from the previous
// chunk's window of the same candidate (one warp per chunk).
__global__ void __launch_bounds__(TPB) k_anchor(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  const int lane = threadIdx.x & 31;
  const int c = (int)((blockIdx.x * (long long)TPB + threadIdx.x) >> 5) + 1;
  if (c >= T) return;
  const long long E0 = x.bs->E0, s0 = x.bs->s_start, q0 = x.st->q;
  const int nc = x.st->geo ? NCAND : NLIN;   // geometric candidates only after an unsettled batch
  const long long a = chunk_warm_start(x, E0, c);
  const long long Jc = a - 1;
  const long long ap = c == 1 ? E0 : chunk_warm_start(x, E0, c - 1);
  const long long Jp = ap - 1;
  int cp[NCAND], ct[NCAND];
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
}

// chunk 1's left edges [s_start, s_1i) counted by the whole grid (y = candidate)
__global__ void __launch_bounds__(TPB) k_anchor_base(Ctx x) {
  pdl_wait();
  __shared__ int red[2][TPB / 32];
  const long long B = x.bs->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  if (T < 2) return;
  const int i = blockIdx.y;
  if (i >= (x.st->geo ? NCAND : NLIN)) return;
  const long long E0 = x.bs->E0, s0 = x.bs->s_start, q0 = x.st->q;
  const long long a = chunk_warm_start(x, E0, 1);
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
  const int i = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int2 carry = make_int2((int)x.st->npix, (int)x.st->ntiles);
  for (int base = 1; base < T; base += 1024 * PER) {
    const int c0 = base + threadIdx.x * PER;
    int2 v[PER];
    int2 tsum = make_int2(0, 0);
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      v[r] = c0 + r < T ? anc[(long long)(c0 + r) * nc + i] : make_int2(0, 0);
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
      if (c0 + r < T) anc[(long long)(c0 + r) * nc + i] = run;
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
__global__ void __launch_bounds__(TPB) k_fp(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  const int c = blockIdx.x * TPB + threadIdx.x;
  if (c >= T) return;
  const long long E0 = x.bs->E0, s0 = x.bs->s_start, q0 = x.st->q;
  const long long a = chunk_warm_start(x, E0, c);
  if (c == 0 || a == E0) {
    x.lc[c] = a - s0;
    x.lu[c] = 32;
    return;
  }
  const int nc = x.st->geo ? NCAND : NLIN;
  long long lens[NCAND], fs[NCAND];
#pragma unroll 1
  for (int i = 0; i < nc; ++i) {
    const long long len = a - max(s0, a - cand_len(x, q0, i));
    const int2 cnt = x.anc[(long long)c * NCAND + i];
    const long long f = (cnt.x >= 1 && cnt.y >= 1) ? regulate(x, len, cnt.x, cnt.y) - len : -1;
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
  // stays well inside their span (windows clamped at the batch start excepted)
  const bool clamped = len_lo >= 0 && len_hi < 0 && len_lo == a - s0;
  if (!clamped && (L < q0 + c_lin_off[0] / 2 || L > q0 + c_lin_off[NLIN - 1] / 2)) x.st->geo_next = 1;
  x.lc[c] = L;
  x.lu[c] = unit;
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
  if (c >= T) return;
  const long long E0 = x.bs->E0, s0 = x.bs->s_start;
  const long long ac = chunk_warm_start(x, E0, c);
  const long long ap = c == 1 ? E0 : chunk_warm_start(x, E0, c - 1);
  const long long Jc = ac - 1, Jp = ap - 1;
  const long long lcc = x.lc[c], lcp = c == 1 ? 0 : x.lc[c - 1];
  const long long luc = x.lu[c], lup = c == 1 ? 32 : x.lu[c - 1];
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

// One lane per chunk, the warp stepping its lanes' events in lockstep.  Each
// lane starts from the longest candidate window just past the regulator's
// fixed point (a too-long window collapses to the true one within a few
// events), warms up, then runs its own chunk.  Evictions of more than a few
// entries (the first trims of a long start window) are counted by the whole
// warp, 32 ring entries per step.
constexpr unsigned WIN_SOLO = 384;   // evictions a lane counts alone (longer: the whole warp)

__global__ void __launch_bounds__(128) k_window_run(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  const int c = blockIdx.x * 128 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if ((blockIdx.x * 128 + (threadIdx.x & ~31)) >= T) return;   // whole warp out of range
  const bool valid = c < T;
  const DevState s = *x.st;
  const long long E0 = x.bs->E0;
  const long long s_start0 = x.bs->s_start;
  const long long b = E0 + (long long)c * x.chunk;
  const long long e = valid ? min(E0 + B, b + x.chunk) : b;
  const long long a = valid ? chunk_warm_start(x, E0, c) : b;
  WState w{0, 1, 0, 0, 0};
  if (valid) {
    if (a == E0) {
      w.s = s_start0;
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
        if (cnt.x >= 1 && cnt.y >= 1 && regulate(x, len, cnt.x, cnt.y) >= len) jstar = j;
      }
      const int g = jstar + 1 < NFINE ? jstar + 1 : NFINE - 1;
      const int2 cnt = x.anc2[(long long)c * NFINE + g];
      w.s = fine_start(x, s_start0, a, center, unit, g);
      w.npix = cnt.x;
      w.ntiles = cnt.y;
      const long long len = a - w.s;
      w.q = (cnt.x >= 1 && cnt.y >= 1) ? regulate(x, len, cnt.x, cnt.y) : len;
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
  // within B + window of it); ring slots as (slot of s_start + offset) & Rm
  const long long base = s_start0;
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
      for (unsigned k = lo; k < hi; ++k) {
        const uint2 rr = x.rnext[(bslot + k) & rm];
        const unsigned dd = jr - k;
        np -= rr.x > dd;
        nt -= rr.y > dd;
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
      if (jr >= br) x.S[jr - e0r] = sr;
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

// Verify chunk boundaries: a chunk is exact once its speculative start state
// equals its predecessor's end state and the predecessor is exact.  Rounds
// re-run, in parallel, every chunk whose start disagrees with its
// predecessor's current end (read before the round writes anything), until
// every boundary agrees; each round makes at least the first disagreeing
// chunk exact.  Then publish the batch's final window state.
__global__ void __launch_bounds__(1024) k_window_fix(Ctx x) {
  pdl_wait();
  __shared__ int n_bad;
  __shared__ long long red_lo[32], red_hi[32];
  const long long B = x.bs->B;
  const int T = (int)((B + x.chunk - 1) / x.chunk);
  const long long E0 = x.bs->E0, s_start = x.bs->s_start;
  int rounds = 0, reruns = 0;
  while (true) {
    if (threadIdx.x == 0) n_bad = 0;
    __syncthreads();
    // each thread owns chunks threadIdx.x + 1024*i; snapshot predecessors first
    constexpr int MAXC = 64;
    int mine[MAXC];
    ChunkRec pre[1];
    int nm = 0;
    for (int c = 1 + threadIdx.x; c < T && nm < MAXC; c += 1024) {
      const ChunkRec &p = x.ch[c - 1];
      const ChunkRec &q = x.ch[c];
      if (q.st_s != p.en_s || q.st_q != p.en_q) mine[nm++] = c;
    }
    if (nm) atomicAdd(&n_bad, nm);
    __syncthreads();
    if (n_bad == 0) break;
    // read every rerun's start state before any write of this round
    long long ss[MAXC], sq[MAXC], snp[MAXC], snt[MAXC], sev[MAXC];
    (void)pre;
    for (int i = 0; i < nm; ++i) {
      const ChunkRec &p = x.ch[mine[i] - 1];
      ss[i] = p.en_s;
      sq[i] = p.en_q;
      snp[i] = p.en_np;
      snt[i] = p.en_nt;
      sev[i] = p.en_ev;
    }
    __syncthreads();
    for (int i = 0; i < nm; ++i) {
      const int m = mine[i];
      WState w{ss[i], sq[i], snp[i], snt[i], sev[i]};
      long long qlo = 0x7FFFFFFFFFFFFFFFLL, qhi = -1;
      const long long b = E0 + (long long)m * x.chunk;
      const long long e = min(E0 + B, b + x.chunk);
      run_window(x, w, b, e, E0, s_start, true, qlo, qhi);
      ChunkRec r;
      r.st_s = ss[i];
      r.st_q = sq[i];
      r.en_s = w.s;
      r.en_q = w.q;
      r.en_np = w.npix;
      r.en_nt = w.ntiles;
      r.en_ev = w.evctr;
      r.qlo = qlo;
      r.qhi = qhi;
      x.ch[m] = r;
    }
    reruns += nm;
    ++rounds;
    __threadfence_block();
    __syncthreads();
  }
  long long lo = 0x7FFFFFFFFFFFFFFFLL, hi = -1;
  for (int c = threadIdx.x; c < T; c += 1024) {
    lo = min(lo, x.ch[c].qlo);
    hi = max(hi, x.ch[c].qhi);
  }
  int rr = __reduce_add_sync(0xffffffffu, reruns);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red_lo[threadIdx.x >> 5] = lo;
    red_hi[threadIdx.x >> 5] = hi;
    if (rr) atomicAdd((unsigned long long *)&x.st->mismatch, (unsigned long long)rr);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < 32; ++w) {
      lo = min(lo, red_lo[w]);
      hi = max(hi, red_hi[w]);
    }
    DevState *s = x.st;
    if (T > 0) {
      const ChunkRec &r = x.ch[T - 1];
      s->s = r.en_s;
      s->q = r.en_q;
      s->npix = r.en_np;
      s->ntiles = r.en_nt;
      s->evctr = r.en_ev;
      if (hi >= 0) {
        s->qtmin = min(s->qtmin, lo);
        s->qtmax = max(s->qtmax, hi);
      }
      s->pops += r.en_s - s_start;
      x.bs->npop = r.en_s - s_start;
    } else {
      x.bs->npop = 0;
    }
    s->chunks += T;
    s->fix_rounds += rounds;
  }
}

// ----------------------------------------------------------------- stale ---

// Every window entry popped in this batch becomes an item, in pop order (the
// order the reference blurs them, _kernels.py:152-189).  An entry is stale iff
// its pixel has no later event up to the popping event.
__global__ void __launch_bounds__(TPB) k_popj(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const long long E0 = x.bs->E0, s_start = x.bs->s_start;
  const unsigned npop = B > 0 ? x.S[B - 1] : 0u;
  const unsigned p = blockIdx.x * TPB + threadIdx.x;   // one thread per eviction (balanced)
  unsigned nst = 0;
  if (p < npop) {
    // popping event: the first jj with S[jj] > p (S is non-decreasing)
    unsigned lo = 0, hi = (unsigned)B - 1;
    while (lo < hi) {
      const unsigned mid = (lo + hi) >> 1;
      if (__ldg(&x.S[mid]) > p) hi = mid; else lo = mid + 1;
    }
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
        if ((unsigned long long)x.rnext[(unsigned long long)k & x.Rm].x > (unsigned long long)(E0 + B - 1 - k))
          it.pad |= ITEM_CARRIED_ONLY;
      }
      ++nst;
    }
    x.item[p] = it;
  }
  nst = __reduce_add_sync(0xffffffffu, nst);
  if ((threadIdx.x & 31) == 0 && nst) atomicAdd((unsigned long long *)&x.bs->stale_batch, (unsigned long long)nst);
}

// -------------------------------------------------------------- temporal ---

// Per sorted position, fully parallel: the event's polarity gathered into
// sorted order and (filter ON) whether the event is evicted stale in this
// batch -- the random loads the serial per-pixel replay would otherwise wait on.
__global__ void __launch_bounds__(TPB) k_posinfo(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const long long i = (long long)blockIdx.x * TPB + threadIdx.x;
  if (i >= B) return;
  const unsigned jj = x.sidx[i];
  x.spol[i] = x.epol[jj];
  if (!x.spatial) return;
  const long long E0 = x.bs->E0, s_start = x.bs->s_start;
  const long long s_end = s_start + x.S[B - 1];
  const long long e = E0 + jj;
  unsigned bidx = FIBAR_NONE;
  if (e < s_end) {
    const unsigned q = (unsigned)(e - s_start);
    if (x.item[q].pix != FIBAR_NONE) bidx = q;
  }
  *reinterpret_cast<uint2 *>(&x.posrec[i]) = make_uint2(jj, bidx);
}

// One thread per pixel segment replays its events in stream order with the
// reference's float32 operation order (_kernels.py:67-73 / 124-130).  Inputs
// are read GROUP positions at a time (all loads issued before the dependent
// arithmetic), so long segments (hot pixels) run at the arithmetic chain's speed.
constexpr int GROUP = 8;
constexpr int LONG_SEG = 512;    // segments longer than this go to k_temporal_long
constexpr int MAX_LONG = 16384;

__global__ void __launch_bounds__(TPB) k_temporal(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const long long i = (long long)blockIdx.x * TPB + threadIdx.x;
  if (i >= B) return;
  const unsigned key = x.skey[i];
  if (i > 0 && x.skey[i - 1] == key) return;
  const unsigned c = x.ekey[x.sidx[i]];
  const long long end = x.spatial ? (long long)x.pt[c].end : -1;
  if (i + LONG_SEG < B && x.skey[i + LONG_SEG] == key) {   // long segment: the warp-parallel kernel
    const unsigned slot = atomicAdd(&x.bs->nlong, 1u);
    if (slot < MAX_LONG) x.longseg[slot] = make_uint2((unsigned)i, c);
    return;
  }
  float pb = x.pbar[c], lv = x.l[c];
  const float g = x.use_gain ? x.gain[c] : 1.0f;
  long long pos = i;
  bool more = true;
  while (more) {
    int8_t pol[GROUP];
    bool in[GROUP];
#pragma unroll
    for (int u = 0; u < GROUP; ++u) {
      const long long q = pos + u;
      in[u] = q < B && (end >= 0 ? q < end : x.skey[q] == key);
      pol[u] = in[u] ? x.spol[q] : (int8_t)0;
    }
#pragma unroll
    for (int u = 0; u < GROUP; ++u) {
      if (!in[u]) {
        more = false;
        break;
      }
      const float p = (float)pol[u];
      pb = faddr(fmulr(x.alpha, pb), fmulr(x.oma, p));
      float d = fsubr(p, pb);
      if (x.use_gain) d = fmulr(d, g);
      lv = faddr(fmulr(x.beta, lv), fmulr(x.h, d));
    }
    pos += GROUP;
  }
  x.pbar[c] = pb;
  x.l[c] = lv;
}

// Filter ON: same replay, recording per position the additive term t2 = h*d,
// the brightness assuming no blur (valid until the pixel's first blur in the
// batch), and which blur each position builds on.
__global__ void __launch_bounds__(TPB) k_temporal_runs(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const long long i = (long long)blockIdx.x * TPB + threadIdx.x;
  if (i >= B) return;
  const unsigned key = x.skey[i];
  if (i > 0 && x.skey[i - 1] == key) return;
  const unsigned c = x.ekey[x.sidx[i]];
  const PixRec prc = x.pt[c];
  const long long end = prc.end;
  if (end - i > LONG_SEG) {   // long segment (hot pixel): the warp-parallel kernel
    const unsigned slot = atomicAdd(&x.bs->nlong, 1u);
    if (slot < MAX_LONG) x.longseg[slot] = make_uint2((unsigned)i, c);
    return;
  }
  unsigned carry = prc.carried;
  if (carry != FIBAR_NONE) x.item[carry].runpos = (unsigned)i;
  float pb = x.pbar[c], lv = x.l[c];
  const float g = x.use_gain ? x.gain[c] : 1.0f;
  for (long long pos = i; pos < end; pos += GROUP) {
    int8_t pol[GROUP];
    unsigned bidx[GROUP];
#pragma unroll
    for (int u = 0; u < GROUP; ++u) {
      const long long q = pos + u;
      pol[u] = q < end ? x.spol[q] : (int8_t)0;
      bidx[u] = q < end ? x.posrec[q].bidx : FIBAR_NONE;
    }
#pragma unroll
    for (int u = 0; u < GROUP; ++u) {
      const long long q = pos + u;
      if (q >= end) break;
      const float p = (float)pol[u];
      pb = faddr(fmulr(x.alpha, pb), fmulr(x.oma, p));
      float d = fsubr(p, pb);
      if (x.use_gain) d = fmulr(d, g);
      const float tt = fmulr(x.h, d);
      lv = faddr(fmulr(x.beta, lv), tt);
      x.t2[q] = tt;
      *reinterpret_cast<uint2 *>(&x.posrec[q].runbase) = make_uint2(carry, __float_as_uint(lv));
      if (bidx[u] != FIBAR_NONE) {
        carry = bidx[u];
        if (q + 1 < end) x.item[bidx[u]].runpos = (unsigned)(q + 1);
      }
    }
  }
  x.pbar[c] = pb;
  // last-touch tables for the next batch's links (the blur stage never reads them)
  const long long elast = x.bs->E0 + x.sidx[end - 1];
  x.plast[c] = elast;
  atomicMax(&x.last_tile[key / x.A], elast);
}

// Long pixel segments (hot pixels: thousands of events per batch) replayed by
// a block: lane i takes the i-th piece (at least LONG_PIECE events), starting
// `twarm` events early from a zero state.  The two float32 recurrences are
// contractions (|alpha|, |beta| < 1), so trajectories from different starts
// become bit-identical after ~24*ln2/-ln(max(alpha, beta)) events (~110 at
// t_cut = 40; twarm is 1.6x that); each lane's piece-start state is checked
// against the previous lane's piece-end state and any piece whose start
// differed is replayed serially from the exact state, so the result is exact
// either way.

__device__ __forceinline__ void iir_step(const Ctx &x, float &pb, float &lv, float p, float g, float &tt) {
  pb = faddr(fmulr(x.alpha, pb), fmulr(x.oma, p));
  float d = fsubr(p, pb);
  if (x.use_gain) d = fmulr(d, g);
  tt = fmulr(x.h, d);
  lv = faddr(fmulr(x.beta, lv), tt);
}

// replay [q0, q1) from (pb, lv), writing the per-position outputs; inputs are
// loaded GROUP at a time so the chain waits on one load per group
__device__ __forceinline__ void replay_piece(const Ctx &x, long long q0, long long q1, float &pb, float &lv, float g,
                                             bool write) {
  for (long long q = q0; q < q1; q += GROUP) {
    int8_t pol[GROUP];
#pragma unroll
    for (int u = 0; u < GROUP; ++u) pol[u] = q + u < q1 ? x.spol[q + u] : (int8_t)0;
#pragma unroll
    for (int u = 0; u < GROUP; ++u) {
      if (q + u >= q1) break;
      float tt;
      iir_step(x, pb, lv, (float)pol[u], g, tt);
      if (write && x.spatial) {
        x.t2[q + u] = tt;
        x.posrec[q + u].val = lv;
      }
    }
  }
}

constexpr int LONG_TPB = 256;      // lanes per long segment (one block)
constexpr int LONG_PIECE = 64;     // minimum events per lane before more lanes join

__global__ void __launch_bounds__(LONG_TPB) k_temporal_long(Ctx x) {
  pdl_wait();
  __shared__ float s_spb[LONG_TPB], s_slv[LONG_TPB], s_epb[LONG_TPB], s_elv[LONG_TPB];
  __shared__ unsigned s_last[LONG_TPB];
  __shared__ int s_bad;
  const unsigned n = min(x.bs->nlong, (unsigned)MAX_LONG);
  const int tid = threadIdx.x;
  for (unsigned sidx = blockIdx.x; sidx < n; sidx += gridDim.x) {
    const uint2 ls = x.longseg[sidx];
    const long long st = ls.x;
    const unsigned c = ls.y;
    long long end;
    if (x.spatial) {
      end = x.pt[c].end;
    } else {
      // segment end by search on the sorted keys (OFF path has no pixel table)
      const unsigned key = x.skey[st];
      long long lo = st + 1, hi = x.bs->B;
      while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (x.skey[mid] == key) lo = mid + 1; else hi = mid;
      }
      end = lo;
    }
    const long long len = end - st;
    const int lanes = (int)min((long long)LONG_TPB, max(32LL, len / LONG_PIECE));
    const long long P = (len + lanes - 1) / lanes;
    const bool on = tid < lanes;
    const long long q0 = on ? min(end, st + tid * P) : end, q1 = on ? min(end, q0 + P) : end;
    const float g = x.use_gain ? x.gain[c] : 1.0f;
    float pb = 0.0f, lv = 0.0f;
    if (tid == 0) {
      pb = x.pbar[c];
      lv = x.l[c];
    } else if (on) {
      replay_piece(x, max(st, q0 - (long long)x.twarm), q0, pb, lv, g, false);
    }
    s_spb[tid] = pb;   // speculative state at the piece start
    s_slv[tid] = lv;
    replay_piece(x, q0, q1, pb, lv, g, true);
    s_epb[tid] = pb;
    s_elv[tid] = lv;
    if (tid == 0) s_bad = 0;
    __syncthreads();
    // verify every boundary; in the rare case a start was wrong, re-run the
    // pieces from there on serially in lane order from the exact states
    if (on && tid > 0 && (__float_as_uint(s_spb[tid]) != __float_as_uint(s_epb[tid - 1]) ||
                          __float_as_uint(s_slv[tid]) != __float_as_uint(s_elv[tid - 1])))
      atomicMax(&s_bad, 1);
    __syncthreads();
    if (s_bad) {
      for (int i = 1; i < lanes; ++i) {
        if (tid == i && (__float_as_uint(s_spb[i]) != __float_as_uint(s_epb[i - 1]) ||
                         __float_as_uint(s_slv[i]) != __float_as_uint(s_elv[i - 1]))) {
          pb = s_epb[i - 1];
          lv = s_elv[i - 1];
          s_spb[i] = pb;
          s_slv[i] = lv;
          replay_piece(x, q0, q1, pb, lv, g, true);
          s_epb[i] = pb;
          s_elv[i] = lv;
        }
        __syncthreads();
      }
    }
    const float fpb = s_epb[lanes - 1], flv = s_elv[lanes - 1];
    if (!x.spatial) {
      if (tid == 0) {
        x.pbar[c] = fpb;
        x.l[c] = flv;
      }
      __syncthreads();
      continue;
    }
    if (tid == 0) {
      x.pbar[c] = fpb;
      const long long elast = x.bs->E0 + x.sidx[end - 1];
      x.plast[c] = elast;
      atomicMax(&x.last_tile[x.skey[st] / x.A], elast);
    }
    // blur bookkeeping: which blur each position builds on (last stale event
    // before it in the segment, or the pixel's carried blur)
    unsigned last = FIBAR_NONE;
    for (long long q = q0; q < q1; q += GROUP) {
      unsigned bidx[GROUP];
#pragma unroll
      for (int u = 0; u < GROUP; ++u) bidx[u] = q + u < q1 ? x.posrec[q + u].bidx : FIBAR_NONE;
#pragma unroll
      for (int u = 0; u < GROUP; ++u) {
        if (bidx[u] != FIBAR_NONE) {
          last = bidx[u];
          if (q + u + 1 < end) x.item[bidx[u]].runpos = (unsigned)(q + u + 1);
        }
      }
    }
    s_last[tid] = last;
    const unsigned carried = x.pt[c].carried;
    if (tid == 0 && carried != FIBAR_NONE) x.item[carried].runpos = (unsigned)st;
    __syncthreads();
    // exclusive "last non-NONE before me" over the lanes: a short backwards scan
    unsigned carry = carried;
    for (int i = tid - 1; i >= 0; --i) {
      if (s_last[i] != FIBAR_NONE) {
        carry = s_last[i];
        break;
      }
    }
    for (long long q = q0; q < q1; q += GROUP) {
      unsigned bidx[GROUP];
#pragma unroll
      for (int u = 0; u < GROUP; ++u) bidx[u] = q + u < q1 ? x.posrec[q + u].bidx : FIBAR_NONE;
#pragma unroll
      for (int u = 0; u < GROUP; ++u) {
        if (q + u >= q1) break;
        x.posrec[q + u].runbase = carry;
        if (bidx[u] != FIBAR_NONE) carry = bidx[u];
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------- blur ---

struct BatchScalars {
  long long E0, B, s_start, s_end;
  unsigned epoch;
};

__device__ __forceinline__ BatchScalars load_bs(const Ctx &x) {
  BatchScalars b;
  b.E0 = x.bs->E0;
  b.B = x.bs->B;
  b.s_start = x.bs->s_start;
  b.s_end = b.s_start + x.bs->npop;
  b.epoch = x.bs->epoch;
  return b;
}

// First resolution of item p's 3x3 taps (_kernels.py:174-188 tap order).  A
// tap's brightness "at item p" is the neighbour's value after every temporal
// update up to the popping event and every earlier blur.  It comes from the
// pixel record (batch segment, carried blur) and the position record of the
// neighbour's latest event at that time: directly (batch-start value or
// first-run value) or, when a blur produced it, after that blur's flag.
// Runs for all items in parallel, before any blur (no waiting).
__global__ void __launch_bounds__(TPB, 4) k_blur_prep(Ctx x) {
  pdl_wait();
  const BatchScalars b = load_bs(x);
  const unsigned npop = (unsigned)(b.s_end - b.s_start);
  const unsigned p = blockIdx.x * TPB + threadIdx.x;
  if (p >= npop) return;
  const Item it = x.item[p];
  BlurPrep out;
  out.okm = 0;
  out.pend = 0;
  if (it.pix == FIBAR_NONE) {
    x.prep[p].okm = 0;
    return;
  }
  const unsigned jrel = it.jrel;
  const int cx = (int)(it.pix % (unsigned)x.W), cy = (int)(it.pix / (unsigned)x.W);
  unsigned nidx[9];
  uint4 pr[9];   // (st, end, carried, -) of each tap's pixel record
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int yy = cy + t / 3 - 1, xx = cx + t % 3 - 1;
    const bool ok = yy >= 0 && yy < x.H && xx >= 0 && xx < x.W;
    nidx[t] = ok ? (unsigned)yy * x.W + xx : it.pix;
    out.okm |= (unsigned)ok << t;
    pr[t] = __ldcg(reinterpret_cast<const uint4 *>(&x.pt[nidx[t]]));
  }
  unsigned posi[9], first[9], last[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    first[t] = last[t] = 0xFFFFFFFFu;
    if (pr[t].y > pr[t].x) {
      first[t] = __ldg(&x.sidx[pr[t].x]);
      last[t] = __ldg(&x.sidx[pr[t].y - 1]);
    }
  }
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    posi[t] = FIBAR_NONE;
    if (pr[t].y <= pr[t].x || first[t] > jrel) continue;
    if (last[t] <= jrel) {
      posi[t] = pr[t].y - 1;
    } else {
      unsigned lo = pr[t].x + 1, hi = pr[t].y - 1;   // answer in [st, end-2]
      while (lo < hi) {
        const unsigned mid = (lo + hi) >> 1;
        if (__ldg(&x.sidx[mid]) <= jrel) lo = mid + 1; else hi = mid;
      }
      posi[t] = lo - 1;
    }
  }
  PosRec rec[9];
#pragma unroll
  for (int t = 0; t < 9; ++t)
    if (posi[t] != FIBAR_NONE) rec[t] = x.posrec[posi[t]];
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    out.val[t] = 0u;
    if (!((out.okm >> t) & 1)) continue;
    bool wait = true;
    if (posi[t] == FIBAR_NONE) {
      if (pr[t].z < p) {                    // blurred (carried) before this item
        out.val[t] = pr[t].z;
      } else {
        out.val[t] = __float_as_uint(x.l[nidx[t]]);
        wait = false;
      }
    } else if (rec[t].bidx < p) {           // its own blur came first
      out.val[t] = rec[t].bidx;
    } else if (rec[t].runbase == FIBAR_NONE) {
      out.val[t] = __float_as_uint(rec[t].val);   // first run: no blur involved
      wait = false;
    } else {                                // rebuilt from blur runbase
      out.val[t] = posi[t] | 0x80000000u;
    }
    if (wait) out.pend |= 1u << t;
  }
  out.runpos = it.runpos;
  x.prep[p] = out;
}

// after blur p of pixel c: brightness of c's following events (up to and
// including its next blurred event) is rebuilt from the blurred value

// after blur p of pixel c: brightness of c's following events (up to and
// including its next blurred event) is rebuilt from the blurred value
__device__ __forceinline__ void materialise_run(const Ctx &x, const BatchScalars &b, unsigned p, unsigned r,
                                                float v) {
  // run positions and their terms are fetched four at a time, so a run costs
  // one round trip per four positions instead of one per position
  while (r < b.B) {
    unsigned rb[4];
    float tt[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool in = r + u < b.B;
      rb[u] = in ? x.posrec[r + u].runbase : FIBAR_NONE;
      tt[u] = in ? x.t2[r + u] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (rb[u] != p) return;
      v = faddr(fmulr(x.beta, v), tt[u]);
      x.posrec[r + u].val = v;
      st_relaxed_u64(&x.mv64[r + u], ((unsigned long long)b.epoch << 32) | __float_as_uint(v));
    }
    r += 4;
  }
}

// Persistent dataflow over the eviction items.  Idle lanes take new items in
// pop order from a global ticket (one warp-aggregated atomic), so every
// dependency -- always an earlier item -- is held by a lane that is already
// running; a waiting lane re-polls the pending flags its prep record left
// open.  The blurred value is published (ready) before the
// pixel's following run is rebuilt (mready).
__global__ void __launch_bounds__(TPB) k_blur(Ctx x) {
  pdl_wait();
  const BatchScalars b = load_bs(x);
  const unsigned npop = (unsigned)(b.s_end - b.s_start);
  const int lane = threadIdx.x & 31;
  unsigned p = FIBAR_NONE, okm = 0, pend = 0, runpos = FIBAR_NONE;
  unsigned val[9];
  bool exhausted = false;
  // the warp draws 32 items at a time from the global ticket and hands them
  // to its free lanes in order (one contended atomic per 32 items); every
  // item below a lane's is taken, so the deadlock-freedom argument holds
  unsigned wbase = 0, wused = 32;
  while (true) {
    unsigned want = __ballot_sync(0xffffffffu, p == FIBAR_NONE && !exhausted);
    while (want) {
      if (wused == 32) {
        unsigned nb = 0;
        if (lane == 0) nb = atomicAdd(&x.bs->ticket, 32u);
        wbase = __shfl_sync(0xffffffffu, nb, 0);
        wused = 0;
      }
      const unsigned take = min((unsigned)__popc(want), 32u - wused);
      const unsigned rank = __popc(want & ((1u << lane) - 1u));
      const bool mine = ((want >> lane) & 1) && rank < take;
      const unsigned q = wbase + wused + rank;
      wused += take;
      want &= ~__ballot_sync(0xffffffffu, mine);
      if (mine) {
        if (q >= npop) {
          exhausted = true;
        } else {
          const uint4 *rec = reinterpret_cast<const uint4 *>(&x.prep[q]);
          const uint4 n0 = __ldcg(rec);
          okm = n0.x;
          if (okm) {
            const uint4 n1 = __ldcg(rec + 1), n2 = __ldcg(rec + 2);
            p = q;
            pend = n0.y;
            val[0] = n0.z;
            val[1] = n0.w;
            val[2] = n1.x;
            val[3] = n1.y;
            val[4] = n1.z;
            val[5] = n1.w;
            val[6] = n2.x;
            val[7] = n2.y;
            val[8] = n2.z;
            runpos = n2.w;
          }
        }
      }
    }
    if (p != FIBAR_NONE) {
      // every open tap polls its value word (epoch | float bits) with an
      // independent relaxed 64-bit load: a matching epoch means the value is
      // there, so no flag/value ordering (and no fence) is involved
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        if (!((pend >> t) & 1)) continue;
        const unsigned s = val[t];
        const unsigned long long w = ld_relaxed_u64((s & 0x80000000u) ? &x.mv64[s & 0x7FFFFFFFu] : &x.bv64[s]);
        if ((unsigned)(w >> 32) != b.epoch) continue;
        val[t] = (unsigned)w;
        pend &= ~(1u << t);
      }
      if (pend == 0) {
        float num = 0.0f, den = 0.0f;
#pragma unroll
        for (int t = 0; t < 9; ++t) {
          if (!((okm >> t) & 1)) continue;
          const float w = (float)((t / 3 == 1 ? 2 : 1) * (t % 3 == 1 ? 2 : 1));
          num = faddr(num, fmulr(w, __uint_as_float(val[t])));
          den = faddr(den, w);
        }
        const float v = __fdiv_rn(num, den);
        st_relaxed_u64(&x.bv64[p], ((unsigned long long)b.epoch << 32) | __float_as_uint(v));
        if (x.dbg_t) {
          unsigned long long tt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
          x.dbg_t[p] = tt;
        }
        if (runpos != FIBAR_NONE) materialise_run(x, b, p, runpos, v);
        p = FIBAR_NONE;
      } else if (x.blur_sleep) {
        __nanosleep(x.blur_sleep);
      }
    }
    if (__all_sync(0xffffffffu, exhausted && p == FIBAR_NONE)) break;
  }
}

// ------------------------------------------------------------------ final ---

__global__ void __launch_bounds__(TPB) k_final(Ctx x) {
  pdl_wait();
  const BatchScalars b = load_bs(x);
  const long long npop = b.s_end - b.s_start;
  const long long total = b.B + npop;
  for (long long idx = (long long)blockIdx.x * TPB + threadIdx.x; idx < total; idx += (long long)gridDim.x * TPB) {
    if (idx < b.B) {
      const long long pos = idx;
      if (pos + 1 < b.B && x.skey[pos + 1] == x.skey[pos]) continue;   // segment tails only
      const PosRec f = x.posrec[pos];
      const unsigned c = x.ekey[f.jj];
      const long long e = b.E0 + f.jj;
      float v = f.val;
      if (x.blur_on && f.bidx != FIBAR_NONE) v = __uint_as_float((unsigned)x.bv64[f.bidx]);
      x.l[c] = v;
      PixRec nr;
      nr.st = 0;
      nr.end = 0;
      nr.carried = FIBAR_NONE;
      nr.pad0 = 0;
      x.pt[c] = nr;
      (void)e;
    } else {
      const unsigned p = (unsigned)(idx - b.B);
      const Item it = x.item[p];
      if (it.pad & ITEM_CARRIED_ONLY) {
        // carried stale entry whose pixel has no events in this batch: the
        // blur is the pixel's only update (segment pixels are finished above)
        if (x.blur_on) x.l[it.pix] = __uint_as_float((unsigned)x.bv64[p]);
        x.pt[it.pix].carried = FIBAR_NONE;
      }
    }
  }
}

__global__ void k_batch_end(Ctx x) {
  pdl_wait();
  DevState *s = x.st;
  const BatchState *bsp = x.bs;
  if (x.spatial && bsp->B > 0) {
    s->geo = s->geo_next;
    s->geo_next = 0;
  }
  s->E += bsp->B;
  if (x.spatial) {
    s->stale += bsp->stale_batch;
    if (x.blur_on) s->blur += bsp->stale_batch;
  }
}

// ---------------------------------------------------------------- read-out ---

__device__ __forceinline__ unsigned order_key(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float order_unkey(unsigned k) {
  const unsigned u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(u);
}

__device__ void sel_bounds(SelState *sel, double g_lo, double g_hi, int mode, double fixed_bound);

// One pass of an exact radix select (digits 11/11/10 bits, MSB first): each
// block histograms the candidates' next digit, and the last block to finish
// picks the digits from the totals (and after the last pass, the bounds).
__global__ void __launch_bounds__(TPB) k_sel_hist(const float *__restrict__ l, long long n, SelState *sel, int pass,
                                                  double g_lo, double g_hi) {
  pdl_wait();
  __shared__ unsigned h[4][2048];
  const int shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
  const unsigned dmask = pass == 2 ? 1023u : 2047u;
  const unsigned hmask = pass == 0 ? 0u : (pass == 1 ? 0xFFE00000u : 0xFFFFFC00u);
  unsigned pref[4];
  bool act[4];
  for (int t = 0; t < 4; ++t) {
    pref[t] = sel->prefix[t];
    act[t] = true;
    for (int u = 0; u < t; ++u)
      if (pref[u] == pref[t]) act[t] = false;
  }
  for (int i = threadIdx.x; i < 4 * 2048; i += TPB) (&h[0][0])[i] = 0;
  __syncthreads();
  // brightness values cluster in a few top digits, so equal digits within a
  // warp are combined first (one shared atomic per distinct digit and target)
  const long long stride = (long long)gridDim.x * TPB;
  const long long n_round = (n + 31) & ~31LL;
  for (long long i = (long long)blockIdx.x * TPB + threadIdx.x; i < n_round; i += stride) {
    const bool in = i < n;
    const unsigned k = in ? order_key(l[i]) : 0u;
    const unsigned d = (k >> shift) & dmask;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (!act[t]) continue;   // warp-uniform
      const bool mine = in && (k & hmask) == pref[t];
      const unsigned key = mine ? d : 0xFFFFFFFFu;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      if (mine && (threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&h[t][d], (unsigned)__popc(peers));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 2048; i += TPB) {
    const unsigned v = (&h[0][0])[i];
    if (v) atomicAdd(&(&sel->hist[0][0])[i], v);
  }
  __threadfence();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(&sel->done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // totals into shared memory (and the global table cleared for the next pass)
  for (int i = threadIdx.x; i < 4 * 2048; i += TPB) {
    (&h[0][0])[i] = __ldcg(&(&sel->hist[0][0])[i]);
    (&sel->hist[0][0])[i] = 0u;
  }
  __syncthreads();
  // one warp per target: the digit holding its remaining rank
  const int t = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nd = pass == 2 ? 1024 : 2048;
  unsigned found_d = 0, found_before = 0, rank = 0;
  if (t < 4) {
    int src = t;
    for (int u = 0; u < t; ++u)
      if (pref[u] == pref[t]) {
        src = u;
        break;
      }
    rank = sel->rank[t];
    unsigned run = 0;
    for (int base = 0; base < nd; base += 32) {
      const unsigned v = h[src][base + lane];
      unsigned inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned tt = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += tt;
      }
      const unsigned excl = run + inc - v;
      const unsigned m = __ballot_sync(0xffffffffu, rank >= excl && rank < run + inc);
      if (m) {
        const int L = __ffs(m) - 1;
        found_d = base + L;
        found_before = __shfl_sync(0xffffffffu, excl, L);
        break;
      }
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  if (t < 4 && lane == 0) {
    sel->prefix[t] = pref[t] | (found_d << shift);
    sel->rank[t] = rank - found_before;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    sel->done = 0;
    if (pass == 2) {
      __threadfence_block();
      sel_bounds(sel, g_lo, g_hi, FIBAR_RENDER_ROBUST, 0.0);
    }
  }
}

__global__ void k_sel_init(SelState *sel, unsigned r0, unsigned r1, unsigned r2, unsigned r3) {
  pdl_wait();
  for (int t = 0; t < 4; ++t) sel->prefix[t] = 0;
  sel->rank[0] = r0;
  sel->rank[1] = r1;
  sel->rank[2] = r2;
  sel->rank[3] = r3;
}

// lo/hi from the selected order statistics (numpy 'linear' percentile, _lerp)
__device__ void sel_bounds(SelState *sel, double g_lo, double g_hi, int mode, double fixed_bound) {
  double lo, hi;
  if (mode == FIBAR_RENDER_ROBUST) {
    const double a0 = (double)order_unkey(sel->prefix[0]), b0 = (double)order_unkey(sel->prefix[1]);
    const double a1 = (double)order_unkey(sel->prefix[2]), b1 = (double)order_unkey(sel->prefix[3]);
    const double d0 = __dsub_rn(b0, a0), d1 = __dsub_rn(b1, a1);
    lo = g_lo >= 0.5 ? __dsub_rn(b0, __dmul_rn(d0, __dsub_rn(1.0, g_lo))) : __dadd_rn(a0, __dmul_rn(d0, g_lo));
    hi = g_hi >= 0.5 ? __dsub_rn(b1, __dmul_rn(d1, __dsub_rn(1.0, g_hi))) : __dadd_rn(a1, __dmul_rn(d1, g_hi));
  } else {
    lo = -fixed_bound;
    hi = fixed_bound;
  }
  sel->lo = lo;
  sel->hi = hi;
  sel->degenerate = !(hi > lo);
}

__global__ void k_sel_bounds(SelState *sel, double g_lo, double g_hi, int mode, double fixed_bound) {
  pdl_wait();
  sel_bounds(sel, g_lo, g_hi, mode, fixed_bound);
}

// u8 = clip(floor((v - lo) * (255 / (hi - lo)) + 0.5), 0, 255) in float64
// (pipeline.py:582-583); degenerate grids render mid-gray (pipeline.py:578-581)
__global__ void __launch_bounds__(TPB) k_render_map(const float *__restrict__ l, long long n,
                                                     const SelState *__restrict__ sel, uint8_t *__restrict__ out) {
  pdl_wait();
  const double lo = sel->lo, hi = sel->hi;
  const bool deg = sel->degenerate;
  const double scale = deg ? 0.0 : __ddiv_rn(255.0, __dsub_rn(hi, lo));
  for (long long i = (long long)blockIdx.x * TPB + threadIdx.x; i < n; i += (long long)gridDim.x * TPB) {
    uint8_t o = 128;
    if (!deg) {
      const double s = __dmul_rn(__dsub_rn((double)l[i], lo), scale);
      double r = floor(__dadd_rn(s, 0.5));
      r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
      o = (uint8_t)r;
    }
    out[i] = o;
  }
}

// ------------------------------------------------------------ EVF1 decode ---

// EVF1 records (event_io.py:353-369): dt u32 LE | xp u16 (bit 15 polarity,
// bits 0..14 x) | y u16.  Two records per thread through one 16-byte load;
// columns out, per-block dt sums for the timestamp scan, first out-of-bounds
// record index (the container is invalid then: DataError, event_io.py:359-365).
constexpr int EV_PER_THREAD = 2;
constexpr int EV_TILE = TPB * EV_PER_THREAD;

__global__ void __launch_bounds__(TPB) k_evf1_decode(const uint4 *__restrict__ rec2, const uint2 *__restrict__ rec1,
                                                     long long nrec, int W, int H, uint16_t *__restrict__ xo,
                                                     uint16_t *__restrict__ yo, int8_t *__restrict__ po,
                                                     unsigned *__restrict__ dto, unsigned long long *__restrict__ bsum,
                                                     unsigned long long *__restrict__ first_bad) {
  pdl_wait();
  __shared__ unsigned long long ws[TPB / 32];
  const long long i0 = ((long long)blockIdx.x * TPB + threadIdx.x) * EV_PER_THREAD;
  unsigned dt[2] = {0u, 0u};
  unsigned xp[2] = {0u, 0u}, yy[2] = {0u, 0u};
  if (i0 + 1 < nrec) {
    const uint4 v = __ldcs(&rec2[i0 >> 1]);
    dt[0] = v.x;
    xp[0] = v.y & 0xFFFFu;
    yy[0] = v.y >> 16;
    dt[1] = v.z;
    xp[1] = v.w & 0xFFFFu;
    yy[1] = v.w >> 16;
  } else if (i0 < nrec) {
    const uint2 v = rec1[i0];
    dt[0] = v.x;
    xp[0] = v.y & 0xFFFFu;
    yy[0] = v.y >> 16;
  }
  unsigned long long s = 0;
#pragma unroll
  for (int r = 0; r < EV_PER_THREAD; ++r) {
    const long long i = i0 + r;
    if (i >= nrec) break;
    const unsigned xx = xp[r] & 0x7FFFu;
    if (xx >= (unsigned)W || yy[r] >= (unsigned)H) atomicMin(first_bad, (unsigned long long)i);
    xo[i] = (uint16_t)xx;
    yo[i] = (uint16_t)yy[r];
    po[i] = (xp[r] >> 15) ? (int8_t)1 : (int8_t)-1;
    dto[i] = dt[r];
    s += dt[r];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < TPB / 32; ++w) t += ws[w];
    bsum[blockIdx.x] = t;
  }
}

// t = t_base + inclusive prefix sum of dt (numpy cumsum in uint64, then + t_base)
__global__ void __launch_bounds__(1024) k_evf1_block_scan(unsigned long long *bsum, int nb, unsigned long long t_base) {
  pdl_wait();
  // one CTA: exclusive scan of the block sums, seeded with t_base
  __shared__ unsigned long long carry;
  __shared__ unsigned long long wt[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = t_base;
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    const unsigned long long v = i < nb ? bsum[i] : 0ull;
    unsigned long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wt[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      const unsigned long long w = wt[lane];
      unsigned long long wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      wt[lane] = wi - w;
    }
    __syncthreads();
    const unsigned long long ex = carry + wt[wid] + inc - v;
    if (i < nb) bsum[i] = ex;
    __syncthreads();
    if (threadIdx.x == 1023) carry = ex + v;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(TPB) k_evf1_times(const unsigned *__restrict__ dt, long long nrec,
                                                    const unsigned long long *__restrict__ bofs,
                                                    unsigned long long *__restrict__ t) {
  pdl_wait();
  __shared__ unsigned long long ws[TPB / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long i0 = ((long long)blockIdx.x * TPB + threadIdx.x) * EV_PER_THREAD;
  unsigned long long d[EV_PER_THREAD], s = 0;
#pragma unroll
  for (int r = 0; r < EV_PER_THREAD; ++r) {
    d[r] = i0 + r < nrec ? dt[i0 + r] : 0ull;
    s += d[r];
  }
  unsigned long long inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) ws[wid] = inc;
  __syncthreads();
  unsigned long long wofs = 0;
  for (int w = 0; w < wid; ++w) wofs += ws[w];
  unsigned long long run = bofs[blockIdx.x] + wofs + inc - s;
#pragma unroll
  for (int r = 0; r < EV_PER_THREAD; ++r) {
    run += d[r];
    if (i0 + r < nrec) t[i0 + r] = run;
  }
}

// --------------------------------------------------------- state export ---

__global__ void k_active_counts(Ctx x, unsigned *cnt) {
  pdl_wait();
  const long long s = x.st->s, E = x.st->E;
  for (long long k = s + (long long)blockIdx.x * TPB + threadIdx.x; k < E; k += (long long)gridDim.x * TPB)
    atomicAdd(&cnt[x.rkey[(unsigned long long)k & x.Rm]], 1u);
}

__global__ void k_tile_counts(Ctx x, const unsigned *cnt, unsigned *tcnt) {
  pdl_wait();
  for (long long c = (long long)blockIdx.x * TPB + threadIdx.x; c < x.n_pix; c += (long long)gridDim.x * TPB) {
    if (cnt[c] == 0) continue;
    const unsigned xx = (unsigned)(c % x.W), yy = (unsigned)(c / x.W);
    atomicAdd(&tcnt[(yy / x.ts) * x.tiles_x + xx / x.ts], 1u);
  }
}

__global__ void k_ring_xy(Ctx x, uint16_t *qx, uint16_t *qy) {
  pdl_wait();
  const long long E = x.st->E;
  const long long qcap = x.n_pix + 1;
  for (long long t = (long long)blockIdx.x * TPB + threadIdx.x; t < qcap; t += (long long)gridDim.x * TPB) {
    uint16_t ox = 0, oy = 0;
    if (E - 1 >= t) {
      const long long k = t + ((E - 1 - t) / qcap) * qcap;
      const unsigned c = x.rkey[(unsigned long long)k & x.Rm];
      ox = (uint16_t)(c % (unsigned)x.W);
      oy = (uint16_t)(c / (unsigned)x.W);
    }
    qx[t] = ox;
    qy[t] = oy;
  }
}

__global__ void k_init_state(DevState *s, long long q0) {
  pdl_wait();
  memset(s, 0, sizeof(DevState));
  s->geo = 1;
  s->q = q0;
  s->qtmin = q0;
  s->qtmax = q0;
  s->epoch = 1;
}

__global__ void k_fill_ll(long long *p, long long n, long long v) {
  pdl_wait();
  for (long long i = (long long)blockIdx.x * TPB + threadIdx.x; i < n; i += (long long)gridDim.x * TPB) p[i] = v;
}
__global__ void k_init_pt(PixRec *p0, PixRec *p1, long long *plast, long long n) {
  pdl_wait();
  for (long long i = (long long)blockIdx.x * TPB + threadIdx.x; i < n; i += (long long)gridDim.x * TPB) {
    PixRec r;
    r.st = 0;
    r.end = 0;
    r.carried = FIBAR_NONE;
    r.pad0 = 0;
    p0[i] = r;
    p1[i] = r;
    plast[i] = -1;
  }
}

int ceil_log2(long long v) {
  int b = 0;
  while ((1LL << b) < v) ++b;
  return b;
}

}  // namespace

struct GraphEntry {
  long long n;               // batch size the graph was captured for
  long long kernels;         // kernels per replay (the launch counter)
  cudaGraphExec_t exec;
};

struct fibar_engine {
  fibar_config cfg{};
  int W = 0, H = 0, ts = 2, A = 4, tiles_x = 0, tiles_y = 0;
  unsigned band_y0 = 0, full_H = 0;
  long long n_pix = 0, n_tiles = 0;
  long long q0 = 0;
  Launcher L;
  long long Bcap = 0;
  int key_bits = 0;
  long long R = 0;
  bool spatial = true, blur_on = true, use_gain = false;
  DevState *st = nullptr;
  float *pbar = nullptr, *l = nullptr, *gain = nullptr;
  PixRec *pt2[2] = {nullptr, nullptr};
  long long *plast = nullptr;
  unsigned *wcnt = nullptr;
  BatchState *bsd = nullptr;   // [2]
  long long *last_tile = nullptr;
  uint2 *ptt = nullptr;
  unsigned *rkey = nullptr;
  uint2 *rnext = nullptr;
  uint16_t *raw_x = nullptr, *raw_y = nullptr;
  int8_t *raw_p = nullptr;
  unsigned *blockcnt = nullptr;
  unsigned *ekey2[2] = {nullptr, nullptr};
  int8_t *epol = nullptr, *spol = nullptr;
  uint2 *longseg = nullptr;
  unsigned *ka2[2] = {nullptr, nullptr}, *va2[2] = {nullptr, nullptr}, *kb2[2] = {nullptr, nullptr},
           *vb2[2] = {nullptr, nullptr}, *hist = nullptr;
  uint2 *dp = nullptr;
  unsigned *S = nullptr;
  unsigned long long *bv64 = nullptr, *mv64 = nullptr;
  BlurPrep *prep = nullptr;
  Item *item2[2] = {nullptr, nullptr};
  PosRec *posrec2[2] = {nullptr, nullptr};
  float *t2_2[2] = {nullptr, nullptr};
  int2 *anc = nullptr, *anc2 = nullptr;
  long long *lc = nullptr, *lu = nullptr;
  ChunkRec *ch = nullptr;
  SelState *sel = nullptr;
  uint8_t *frame = nullptr;
  unsigned *cnt_tmp = nullptr, *tcnt_tmp = nullptr;
  uint16_t *q_tmp = nullptr;
  // host packets: CPU copy into pinned staging set `cur`, one H2D per batch on
  // a copy stream into device staging set `cur`, double buffered so the copy
  // of batch k+1 overlaps the compute of batch k
  uint16_t *hx[2] = {nullptr, nullptr}, *hy[2] = {nullptr, nullptr};
  int8_t *hp[2] = {nullptr, nullptr};
  uint16_t *sx[2] = {nullptr, nullptr}, *sy[2] = {nullptr, nullptr};
  int8_t *sp_[2] = {nullptr, nullptr};
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  int cur = 0;
  long long hfill = 0;
  const uint16_t *zx = nullptr, *zy = nullptr;  // pending zero-copy device range (contiguous device packets)
  const int8_t *zp = nullptr;
  long long zn = 0;
  long long batches = 0;
  // filter ON: batch k's blur stage (blur_prep, blur, final) runs on bstream
  // while batch k+1's front end runs on the engine stream; per-batch buffers
  // are double buffered by batch parity
  cudaStream_t bstream = nullptr;
  // small batches: one CUDA graph per batch size, fed from fixed input buffers
  bool graphs_on = true;
  cudaStream_t capstream = nullptr;
  long long graph_max = 1LL << 17;
  std::vector<GraphEntry> graphs;
  uint16_t *gx = nullptr, *gy = nullptr;
  int8_t *gp = nullptr;
  int blur_grid_serial = 148;
  cudaEvent_t evF[2] = {nullptr, nullptr}, evB[2] = {nullptr, nullptr};
  int last_b = -1;   // parity of the newest batch with a blur stage in flight
  bool b_used[2] = {false, false};
  int nsm = 148;
  int blur_grid = 148;
  int chunk = 64, warm = 64, debug = 0;
  int twarm = 256;
  bool serial = false;   // FIBAR_SERIAL: blur stage on the engine stream (no overlap; for measurement)
  unsigned blur_sleep = 0;
  unsigned long long *dbg_t = nullptr, *dbg_g = nullptr;

  Ctx ctx(const unsigned *skey, const unsigned *sidx, long long n_raw, int par) const {
    Ctx x{};
    x.W = W;
    x.H = H;
    x.band_y0 = band_y0;
    x.full_H = full_H;
    x.ts = ts;
    x.tiles_x = tiles_x;
    x.A = A;
    x.n_pix = n_pix;
    x.num = cfg.fill_num;
    x.numA = cfg.fill_num * (long long)A;
    x.den = cfg.fill_den;
    x.qmin = cfg.q_min;
    x.qmax = cfg.q_max;
    x.every = cfg.regulate_every;
    x.alpha = cfg.alpha;
    x.oma = cfg.one_m_alpha;
    x.beta = cfg.beta;
    x.h = cfg.half_1p_beta;
    x.use_gain = use_gain;
    x.blur_on = blur_on;
    x.spatial = spatial;
    x.st = st;
    x.pbar = pbar;
    x.l = l;
    x.gain = gain;
    x.pt = pt2[par];
    x.plast = plast;
    x.wcnt = wcnt;
    x.bs = bsd ? bsd + par : nullptr;
    x.last_tile = last_tile;
    x.ptt = ptt;
    x.rkey = rkey;
    x.rnext = rnext;
    x.Rm = (unsigned long long)(R - 1);
    x.raw_x = raw_x;
    x.raw_y = raw_y;
    x.raw_p = raw_p;
    x.n_raw = n_raw;
    x.blockcnt = blockcnt;
    x.ekey = ekey2[par];
    x.epol = epol;
    x.spol = spol;
    x.longseg = longseg;
    x.tkey = ka2[par];
    x.skey = skey;
    x.sidx = sidx;
    x.dp = dp;
    x.S = S;
    x.item = item2[par];
    x.posrec = posrec2[par];
    x.t2 = t2_2[par];
    x.bv64 = bv64;
    x.mv64 = mv64;
    x.prep = prep;
    x.chunk = chunk;
    x.twarm = twarm;
    x.debug = debug;
    x.blur_sleep = blur_sleep;
    x.dbg_t = dbg_t;
    x.dbg_g = dbg_g;
    x.warm = warm;
    x.anc = anc;
    x.anc2 = anc2;
    x.lc = lc;
    x.lu = lu;
    x.ch = ch;
    return x;
  }
};

namespace {

template <class T>
int dalloc(T **p, long long count) {
  if (count <= 0) count = 1;
  cudaError_t e = cudaMalloc((void **)p, sizeof(T) * (size_t)count);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  return 0;
}

// make the engine stream wait for the newest blur stage (before any read)
int join_blur(fibar_engine *g) {
  if (g->last_b >= 0) CK(cudaStreamWaitEvent(g->L.stream, g->evB[g->last_b], 0));
  return 0;
}

int init_state(fibar_engine *g) {
  cudaStream_t s = g->L.stream;
  join_blur(g);
  g->last_b = -1;
  g->b_used[0] = g->b_used[1] = false;
  fibar_launch(g->L, "init", k_init_state, 1, 1, 0, s, g->st, g->q0);
  CK(cudaMemsetAsync(g->pbar, 0, sizeof(float) * g->n_pix, s));
  CK(cudaMemsetAsync(g->l, 0, sizeof(float) * g->n_pix, s));
  if (g->spatial) {
    fibar_launch(g->L, "init", k_init_pt, g->nsm * 4, TPB, 0, s, g->pt2[0], g->pt2[1], g->plast, g->n_pix);
    fibar_launch(g->L, "init", k_fill_ll, g->nsm * 4, TPB, 0, s, g->last_tile, g->n_tiles, -1);
    CK(cudaMemsetAsync(g->rkey, 0, sizeof(unsigned) * g->R, s));
    CK(cudaMemsetAsync(g->wcnt, 0, sizeof(unsigned) * g->n_pix, s));
    CK(cudaMemsetAsync(g->rnext, 0xFF, sizeof(uint2) * g->R, s));
    CK(cudaMemsetAsync(g->bv64, 0, sizeof(unsigned long long) * (g->Bcap + g->n_pix + 2), s));
    CK(cudaMemsetAsync(g->mv64, 0, sizeof(unsigned long long) * g->Bcap, s));
  }
  g->zn = 0;
  g->hfill = 0;
  CK(cudaGetLastError());
  return 0;
}

// Enqueue one device batch.  graph == false: the streamed form (blur stage on
// the second stream, cross-batch events).  graph == true: everything on the
// engine stream with parity-0 buffers and no events, the form captured into a
// CUDA graph for small batches (see run_batch_raw).
int enqueue_batch(fibar_engine *g, const uint16_t *rx0, const uint16_t *ry0, const int8_t *rp0, long long n_raw,
                  cudaEvent_t used_ev, int par, bool graph) {
  Launcher &L = g->L;
  cudaStream_t s = L.stream;
  // this parity's buffers are free once the batch two back finished its blur stage
  if (!graph && g->spatial && g->b_used[par]) CK(cudaStreamWaitEvent(s, g->evB[par], 0));
  const int nb_in = (int)((n_raw + IN_TILE - 1) / IN_TILE);
  Ctx x = g->ctx(nullptr, nullptr, n_raw, par);
  x.raw_x = rx0;
  x.raw_y = ry0;
  x.raw_p = rp0;
  fibar_launch(L, "count_inb", k_count_inb, nb_in, TPB, 0, s, x, nb_in);
  scan_exclusive_u32(L, g->blockcnt, nb_in + 1);
  fibar_launch(L, "compact", k_compact, nb_in, TPB, 0, s, x, nb_in);
  if (used_ev) CK(cudaEventRecord(used_ev, s));   // the raw staging may be refilled from here on
  const int where = radix_sort_pairs(L, g->ka2[par], g->va2[par], g->kb2[par], g->vb2[par], g->hist, &g->bsd[par].B,
                                     n_raw, g->key_bits);
  const unsigned *skey = where ? g->kb2[par] : g->ka2[par];
  const unsigned *sidx = where ? g->vb2[par] : g->va2[par];
  {
    const uint16_t *rx = x.raw_x, *ry = x.raw_y;
    const int8_t *rp = x.raw_p;
    x = g->ctx(skey, sidx, n_raw, par);
    x.raw_x = rx;
    x.raw_y = ry;
    x.raw_p = rp;
  }
  const int nb = (int)((n_raw + TPB - 1) / TPB);
  if (g->spatial) {
    const int T = (int)((n_raw + g->chunk - 1) / g->chunk);
    fibar_launch(L, "seg_marks", k_seg_marks, nb, TPB, 0, s, x);
    fibar_launch(L, "link", k_link, nb, TPB, 0, s, x);
    fibar_launch(L, "anchor", k_anchor, (int)(((long long)T * 32 + TPB - 1) / TPB), TPB, 0, s, x);
    fibar_launch(L, "anchor_base", k_anchor_base, dim3(g->nsm / 2, NCAND), TPB, 0, s, x);
    fibar_launch(L, "anchor_scan", k_anchor_scan, NCAND, 1024, 0, s, x, g->anc, NCAND);
    fibar_launch(L, "fp", k_fp, (T + TPB - 1) / TPB, TPB, 0, s, x);
    fibar_launch(L, "anchor2", k_anchor2, (int)(((long long)T * 32 + TPB - 1) / TPB), TPB, 0, s, x);
    fibar_launch(L, "anchor_scan", k_anchor_scan, NFINE, 1024, 0, s, x, g->anc2, NFINE);
    fibar_launch(L, "window_run", k_window_run, (T + 127) / 128, 128, 0, s, x);
    fibar_launch(L, "window_fix", k_window_fix, 1, 1024, 0, s, x);
    fibar_launch(L, "popj", k_popj, (int)((n_raw + g->n_pix + TPB) / TPB), TPB, 0, s, x);
    fibar_launch(L, "posinfo", k_posinfo, nb, TPB, 0, s, x);
    // the replay reads the brightness the previous batch's blur stage finishes
    if (!graph && g->last_b >= 0) CK(cudaStreamWaitEvent(s, g->evB[g->last_b], 0));
    fibar_launch(L, "temporal", k_temporal_runs, nb, TPB, 0, s, x);
    fibar_launch(L, "temporal_long", k_temporal_long, g->nsm * 2, LONG_TPB, 0, s, x);
    fibar_launch(L, "batch_end", k_batch_end, 1, 1, 0, s, x);
    // blur stage on its own stream: overlaps the next batch's front end
    cudaStream_t bs = (g->serial || graph) ? s : g->bstream;
    if (!graph) {
      CK(cudaEventRecord(g->evF[par], s));
      CK(cudaStreamWaitEvent(bs, g->evF[par], 0));
    }
    L.stream = bs;
    if (g->blur_on) {
      const int nbp = (int)((n_raw + g->n_pix + TPB) / TPB);
      fibar_launch(L, "blur_prep", k_blur_prep, nbp, TPB, 0, bs, x);
      fibar_launch(L, "blur", k_blur, graph ? g->blur_grid_serial : g->blur_grid, TPB, 0, bs, x);
    }
    fibar_launch(L, "final", k_final, g->nsm * 8, TPB, 0, bs, x);
    L.stream = s;
    if (!graph) {
      CK(cudaEventRecord(g->evB[par], bs));
      g->b_used[par] = true;
      g->last_b = par;
    }
  } else {
    fibar_launch(L, "posinfo", k_posinfo, nb, TPB, 0, s, x);
    fibar_launch(L, "temporal", k_temporal, nb, TPB, 0, s, x);
    fibar_launch(L, "temporal_long", k_temporal_long, g->nsm * 2, LONG_TPB, 0, s, x);
    fibar_launch(L, "batch_end", k_batch_end, 1, 1, 0, s, x);
  }
  CK(cudaGetLastError());
  return 0;
}

// A small batch is launch-bound (~45 dependent kernels doing a few us of work
// each), so it runs as one CUDA graph per batch size: its inputs are copied
// into fixed graph buffers, the kernel sequence is captured once per size and
// replayed with a single launch.  Large batches stream (two-stream overlap).
int run_batch_raw(fibar_engine *g, const uint16_t *rx0, const uint16_t *ry0, const int8_t *rp0, long long n_raw,
                  cudaEvent_t used_ev) {
  if (n_raw <= 0) return 0;
  Launcher &L = g->L;
  cudaStream_t s = L.stream;
  if (!g->graphs_on || L.prof || n_raw > g->graph_max) {
    const int par = g->spatial ? (int)(g->batches & 1) : 0;
    int rc = enqueue_batch(g, rx0, ry0, rp0, n_raw, used_ev, par, false);
    if (rc) return rc;
    g->batches++;
    return 0;
  }
  // graph form: after every earlier blur stage (it reuses parity-0 buffers)
  join_blur(g);
  g->last_b = -1;
  g->b_used[0] = g->b_used[1] = false;
  CK(cudaMemcpyAsync(g->gx, rx0, sizeof(uint16_t) * n_raw, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(g->gy, ry0, sizeof(uint16_t) * n_raw, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(g->gp, rp0, sizeof(int8_t) * n_raw, cudaMemcpyDeviceToDevice, s));
  if (used_ev) CK(cudaEventRecord(used_ev, s));   // the raw staging may be refilled from here on
  GraphEntry *hit = nullptr;
  for (auto &ge : g->graphs)
    if (ge.n == n_raw) hit = &ge;
  if (!hit) {
    if (g->graphs.size() >= 8) {   // small cache: drop the oldest size
      cudaGraphExecDestroy(g->graphs.front().exec);
      g->graphs.erase(g->graphs.begin());
    }
    // captured on a private stream (the caller's may be the legacy default
    // stream, which cannot be captured); replayed on the caller's
    cudaGraph_t graph = nullptr;
    const long long l0 = L.launches;
    if (!g->capstream) CK(cudaStreamCreateWithFlags(&g->capstream, cudaStreamNonBlocking));
    cudaError_t ce = cudaStreamBeginCapture(g->capstream, cudaStreamCaptureModeThreadLocal);
    int rc = 0;
    if (ce == cudaSuccess) {
      L.stream = g->capstream;
      rc = enqueue_batch(g, g->gx, g->gy, g->gp, n_raw, nullptr, 0, true);
      L.stream = s;
      ce = cudaStreamEndCapture(g->capstream, &graph);
    }
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    GraphEntry ge;
    ge.n = n_raw;
    ge.kernels = L.launches - l0;
    L.launches = l0;
    if (ce == cudaSuccess) {
      ce = cudaGraphInstantiate(&ge.exec, graph, 0);
      cudaGraphDestroy(graph);
    }
    if (ce != cudaSuccess) {
      // capture not possible here (e.g. the calling thread is itself capturing
      // in global mode): run the same serial schedule without a graph from now on
      cudaGetLastError();
      g->graphs_on = false;
      rc = enqueue_batch(g, g->gx, g->gy, g->gp, n_raw, nullptr, 0, true);
      if (rc) return rc;
      g->batches++;
      return 0;
    }
    g->graphs.push_back(ge);
    hit = &g->graphs.back();
  }
  CK(cudaGraphLaunch(hit->exec, s));
  L.launches += hit->kernels;
  g->batches++;
  return 0;
}

// hand the filled host staging set to the device and run it
// pinned host packets of at least half a device batch skip the CPU staging
// copy (smaller ones are coalesced through the staging buffers as before)
long long direct_min(const fibar_engine *g) { return std::max(1LL << 16, g->Bcap / 2); }

bool is_pinned(const void *ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int launch_host_batch(fibar_engine *g) {
  if (g->hfill == 0) return 0;
  const int c = g->cur;
  const long long n = g->hfill;
  CK(cudaStreamWaitEvent(g->cstream, g->ev_used[c], 0));
  CK(cudaMemcpyAsync(g->sx[c], g->hx[c], sizeof(uint16_t) * n, cudaMemcpyHostToDevice, g->cstream));
  CK(cudaMemcpyAsync(g->sy[c], g->hy[c], sizeof(uint16_t) * n, cudaMemcpyHostToDevice, g->cstream));
  CK(cudaMemcpyAsync(g->sp_[c], g->hp[c], sizeof(int8_t) * n, cudaMemcpyHostToDevice, g->cstream));
  CK(cudaEventRecord(g->ev_h2d[c], g->cstream));
  CK(cudaStreamWaitEvent(g->L.stream, g->ev_h2d[c], 0));
  g->hfill = 0;
  g->cur ^= 1;
  return run_batch_raw(g, g->sx[c], g->sy[c], g->sp_[c], n, g->ev_used[c]);
}

// run everything pending (zero-copy device range, then staged host packets)
int run_batch(fibar_engine *g) {
  if (g->zn > 0) {
    const long long n = g->zn;
    g->zn = 0;
    int rc = run_batch_raw(g, g->zx, g->zy, g->zp, n, nullptr);
    if (rc) return rc;
  }
  return launch_host_batch(g);
}

// run everything pending and order the engine stream after the blur stage
int sync_point(fibar_engine *g) {
  int rc = run_batch(g);
  if (rc) return rc;
  return join_blur(g);
}

// read-out (pipeline.py:562-584) of n float32 values at l: exact order
// statistics for the robust bounds (numpy 'linear' percentile), float64 map
int render_core(Launcher &L, const float *l, long long n, int32_t mode, double fixed_bound, uint8_t *out,
                int32_t out_mem, double *bounds, int32_t *degenerate, SelState *sel, uint8_t *frame, int nsm) {
  if (mode == FIBAR_RENDER_FIXED && !(fixed_bound > 0)) return fail(FIBAR_E_CONFIG, "fixed scale bound must be positive");
  if (mode != FIBAR_RENDER_FIXED && mode != FIBAR_RENDER_ROBUST) return fail(FIBAR_E_CONFIG, "unknown scale mode");
  cudaStream_t s = L.stream;
  double g_lo = 0, g_hi = 0;
  if (mode == FIBAR_RENDER_ROBUST) {
    // virtual index (n-1)*q, neighbours floor / floor+1, clamped at the top
    const double qs[2] = {1.0 / 100.0, 99.0 / 100.0};
    double gam[2];
    unsigned rk[4];
    for (int t = 0; t < 2; ++t) {
      const double v = (double)(n - 1) * qs[t];
      long long prev, next;
      if (v >= (double)(n - 1)) {
        prev = next = n - 1;
        gam[t] = v + 1.0;   // numpy's gamma uses index -1 here; a == b so the value is unaffected
      } else if (v < 0) {
        prev = next = 0;
        gam[t] = v;
      } else {
        prev = (long long)std::floor(v);
        next = prev + 1;
        gam[t] = v - (double)prev;
      }
      rk[2 * t] = (unsigned)prev;
      rk[2 * t + 1] = (unsigned)next;
    }
    g_lo = gam[0];
    g_hi = gam[1];
    fibar_launch(L, "sel_init", k_sel_init, 1, 1, 0, s, sel, rk[0], rk[1], rk[2], rk[3]);
    const int grid = nsm * 2;
    for (int pass = 0; pass < 3; ++pass)
      fibar_launch(L, "sel_hist", k_sel_hist, grid, TPB, 0, s, l, n, sel, pass, g_lo, g_hi);
  } else {
    fibar_launch(L, "sel_bounds", k_sel_bounds, 1, 1, 0, s, sel, g_lo, g_hi, mode, fixed_bound);
  }
  uint8_t *dst = out_mem == FIBAR_MEM_DEVICE ? out : frame;
  fibar_launch(L, "render_map", k_render_map, nsm * 4, TPB, 0, s, l, n, sel, dst);
  CK(cudaGetLastError());
  if (out_mem != FIBAR_MEM_DEVICE) CK(cudaMemcpyAsync(out, frame, n, cudaMemcpyDeviceToHost, s));
  if (bounds || degenerate || out_mem != FIBAR_MEM_DEVICE) {
    struct {
      double lo, hi;
      int degenerate;
    } h;
    CK(cudaMemcpyAsync(&h, &sel->lo, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (bounds) {
      bounds[0] = h.lo;
      bounds[1] = h.hi;
    }
    if (degenerate) *degenerate = h.degenerate;
  }
  return 0;
}

}  // namespace

// ------------------------------------------------------------------ C ABI ---

extern "C" {

const char *fibar_last_error(void) { return g_err.c_str(); }

int fibar_create(const fibar_config *cfg, void *stream, fibar_engine **out) {
  if (!cfg || !out) return fail(FIBAR_E_CONFIG, "null argument");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(FIBAR_E_NODEVICE, "no CUDA device");
  if (cfg->width < 2 || cfg->height < 2) return fail(FIBAR_E_CONFIG, "geometry must be at least 2x2");
  if (cfg->tile_side < 2) return fail(FIBAR_E_CONFIG, "tile_side must be >= 2");
  if (cfg->regulate_every < 1) return fail(FIBAR_E_CONFIG, "regulate_every must be >= 1");
  const long long n = (long long)cfg->width * cfg->height;
  if (cfg->q_max > n) return fail(FIBAR_E_CONFIG, "q_max exceeds pixel count");
  if (cfg->q_min < 1 || cfg->q_min > cfg->q_max) return fail(FIBAR_E_CONFIG, "bad q_min/q_max");
  if (cfg->fill_num < 1 || cfg->fill_den < 1) return fail(FIBAR_E_CONFIG, "bad fill ratio");
  if (cfg->width > 65535 || cfg->height > 65535) return fail(FIBAR_E_CONFIG, "coordinates must fit uint16");
  if (cfg->sensor_height > 0) {
    if (cfg->band_y0 < 0 || cfg->band_y0 + cfg->height > cfg->sensor_height)
      return fail(FIBAR_E_CONFIG, "row band outside the sensor");
    if (cfg->spatial_enabled && (cfg->band_y0 != 0 || cfg->height != cfg->sensor_height))
      return fail(FIBAR_E_CONFIG, "row bands need the spatial filter off (the window is one global FIFO)");
  }
  fibar_engine *g = new fibar_engine();
  g->cfg = *cfg;
  g->cfg.gain = nullptr;
  g->W = cfg->width;
  g->H = cfg->height;
  g->band_y0 = (unsigned)cfg->band_y0;
  g->full_H = cfg->sensor_height > 0 ? (unsigned)cfg->sensor_height : (unsigned)cfg->height;
  g->ts = cfg->tile_side;
  g->A = g->ts * g->ts;
  g->tiles_x = (g->W + g->ts - 1) / g->ts;
  g->tiles_y = (g->H + g->ts - 1) / g->ts;
  g->n_pix = n;
  g->n_tiles = (long long)g->tiles_x * g->tiles_y;
  g->q0 = std::min(std::max(n / 16, (long long)cfg->q_min), (long long)cfg->q_max);
  g->L.stream = (cudaStream_t)stream;
  g->spatial = cfg->spatial_enabled != 0;
  g->blur_on = cfg->blur_enabled != 0;
  g->use_gain = cfg->gain != nullptr;
  g->Bcap = cfg->batch_capacity > 0 ? cfg->batch_capacity : (1LL << 20);
  if (g->Bcap > (1LL << 28)) g->Bcap = 1LL << 28;
  if (g->Bcap < 1024) g->Bcap = std::max(g->Bcap, 16LL);
  g->key_bits = ceil_log2(g->n_tiles * g->A);
  // window-speculation tuning knobs (results never depend on them; the verifier
  // re-runs any chunk whose speculative start was wrong)
  if (const char *v = getenv("FIBAR_CHUNK")) g->chunk = std::max(CHUNK_MIN, atoi(v));
  if (const char *v = getenv("FIBAR_WARM")) g->warm = std::max(0, atoi(v));
  if (const char *v = getenv("FIBAR_DEBUG_WINDOW")) g->debug = atoi(v);
  if (const char *v = getenv("FIBAR_SERIAL")) g->serial = atoi(v) != 0;
  if (const char *v = getenv("FIBAR_PDL")) g->L.pdl = atoi(v) != 0;
  {
    // contraction of the slower recurrence: events until any two float32
    // trajectories agree to the last bit, with a 1.6x margin
    const double r = std::max((double)cfg->alpha, (double)cfg->beta);
    const double steps = (r > 0.0 && r < 1.0) ? 24.0 * std::log(2.0) / -std::log(r) : 1024.0;
    g->twarm = (int)std::min(2048.0, std::max(64.0, std::ceil(1.6 * steps)));
  }
  g->R = 1LL << ceil_log2(n + 1 + g->Bcap);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g->nsm, cudaDevAttrMultiProcessorCount, dev);
  {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_blur, TPB, 0);
    g->blur_grid_serial = g->nsm * std::max(1, std::min(per_sm, 4));   // graph form: nothing to overlap with
    // the blur stage overlaps the next batch's front end: one 256-thread block
    // per SM leaves the rest of each SM to the front end (measured: 1/SM gives
    // 10.2 ms per 10M config-2 events vs 11.2 at 2/SM and 12.6 serialised)
    const int occ = per_sm;
    per_sm = std::min(per_sm, g->serial ? 4 : 1);
    if (const char *v = getenv("FIBAR_BLUR_BLOCKS")) per_sm = std::min(occ, std::max(1, atoi(v)));
    g->blur_grid = g->nsm * std::max(1, per_sm);
    if (const char *v = getenv("FIBAR_BLUR_SLEEP")) g->blur_sleep = (unsigned)atoi(v);
    if (const char *v = getenv("FIBAR_GRAPHS")) g->graphs_on = atoi(v) != 0;
    if (const char *v = getenv("FIBAR_GRAPH_MAX")) g->graph_max = atoll(v);
    g->graph_max = std::min(g->graph_max, g->Bcap);
  }
  int rc = 0;
  const long long Bc = g->Bcap;
  const int nb_in = (int)((Bc + IN_TILE - 1) / IN_TILE);
  const int nb_rs = (int)((Bc + 2047) / 2048);
  const long long T = (Bc + CHUNK_MIN - 1) / CHUNK_MIN + 1;
  const long long npop_cap = Bc + n + 2;
  rc |= dalloc(&g->st, 1);
  rc |= dalloc(&g->pbar, n);
  rc |= dalloc(&g->l, n);
  for (int c = 0; c < 2; ++c) {
    rc |= dalloc(&g->sx[c], Bc);
    rc |= dalloc(&g->sy[c], Bc);
    rc |= dalloc(&g->sp_[c], Bc);
    if (cudaMallocHost((void **)&g->hx[c], sizeof(uint16_t) * Bc) != cudaSuccess ||
        cudaMallocHost((void **)&g->hy[c], sizeof(uint16_t) * Bc) != cudaSuccess ||
        cudaMallocHost((void **)&g->hp[c], sizeof(int8_t) * Bc) != cudaSuccess)
      rc |= fail(FIBAR_E_CUDA, "cudaMallocHost");
    cudaEventCreateWithFlags(&g->ev_h2d[c], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->ev_used[c], cudaEventDisableTiming);
  }
  cudaStreamCreateWithFlags(&g->cstream, cudaStreamNonBlocking);
  rc |= dalloc(&g->blockcnt, nb_in + 1);
  if (g->graphs_on && g->graph_max > 0) {
    rc |= dalloc(&g->gx, g->graph_max);
    rc |= dalloc(&g->gy, g->graph_max);
    rc |= dalloc(&g->gp, g->graph_max);
  }
  rc |= dalloc(&g->epol, Bc);
  rc |= dalloc(&g->spol, Bc);
  rc |= dalloc(&g->longseg, 16384);
  rc |= dalloc(&g->bsd, 2);
  if (!rc) cudaMemset(g->bsd, 0, 2 * sizeof(BatchState));
  for (int c = 0; c < 2; ++c) {
    // the filter-off path runs every batch on one stream: one set suffices
    const bool own = c == 0 || g->spatial;
    if (own) {
      rc |= dalloc(&g->ekey2[c], Bc);
      rc |= dalloc(&g->ka2[c], Bc);
      rc |= dalloc(&g->va2[c], Bc);
      rc |= dalloc(&g->kb2[c], Bc);
      rc |= dalloc(&g->vb2[c], Bc);
    }
  }
  rc |= dalloc(&g->hist, 256LL * nb_rs + 256LL * nb_rs / 4096 + 8);
  rc |= dalloc(&g->sel, 1);
  if (!rc) cudaMemset(g->sel, 0, sizeof(SelState));
  rc |= dalloc(&g->frame, n);
  if (g->use_gain) {
    rc |= dalloc(&g->gain, n);
    if (!rc) cudaMemcpy(g->gain, cfg->gain, sizeof(float) * n, cudaMemcpyHostToDevice);
  }
  if (g->spatial) {
    for (int c = 0; c < 2; ++c) {
      rc |= dalloc(&g->pt2[c], n);
      rc |= dalloc(&g->item2[c], npop_cap);
      rc |= dalloc(&g->t2_2[c], Bc);
      rc |= dalloc(&g->posrec2[c], Bc);
    }
    rc |= dalloc(&g->plast, n);
    rc |= dalloc(&g->wcnt, n);
    {
      // the blur stage is the latency-critical chain: its blocks go first when
      // SM slots free up, the next batch's front end fills the rest
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      if (const char *v = getenv("FIBAR_BLUR_PRIO")) hi = atoi(v) ? hi : lo;
      cudaStreamCreateWithPriority(&g->bstream, cudaStreamNonBlocking, hi);
    }
    for (int c = 0; c < 2; ++c) {
      cudaEventCreateWithFlags(&g->evF[c], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g->evB[c], cudaEventDisableTiming);
    }
    rc |= dalloc(&g->last_tile, g->n_tiles);
    rc |= dalloc(&g->ptt, g->n_tiles);
    rc |= dalloc(&g->rkey, g->R);
    rc |= dalloc(&g->rnext, g->R);
    rc |= dalloc(&g->dp, Bc);
    rc |= dalloc(&g->S, Bc);
    rc |= dalloc(&g->bv64, npop_cap);
    rc |= dalloc(&g->mv64, Bc);
    rc |= dalloc(&g->prep, npop_cap);
    rc |= dalloc(&g->anc, T * NCAND);
    rc |= dalloc(&g->anc2, T * NFINE);
    rc |= dalloc(&g->lc, T);
    rc |= dalloc(&g->lu, T);
    rc |= dalloc(&g->ch, T);
  }
  if (g->spatial && getenv("FIBAR_DEBUG_TIMES")) {
    rc |= dalloc(&g->dbg_t, npop_cap);
    rc |= dalloc(&g->dbg_g, npop_cap);
  }
  if (rc) {
    fibar_destroy(g);
    return rc;
  }
  rc = init_state(g);
  if (rc) {
    fibar_destroy(g);
    return rc;
  }
  *out = g;
  return 0;
}

int fibar_destroy(fibar_engine *g) {
  if (!g) return 0;
  if (g->bstream) cudaStreamSynchronize(g->bstream);
  void *ptrs[] = {g->st, g->pbar, g->l, g->gain, g->plast, g->wcnt, g->bsd, g->last_tile, g->ptt, g->rkey, g->rnext, g->raw_x,
                  g->raw_y, g->raw_p, g->blockcnt, g->epol, g->spol, g->longseg, g->hist,
                  g->dp, g->S, g->bv64, g->mv64, g->prep, g->anc, g->anc2, g->lc, g->lu, g->ch, g->sel, g->frame,
                  g->cnt_tmp, g->tcnt_tmp, g->q_tmp, g->dbg_t, g->dbg_g};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  for (cudaEvent_t ev : g->L.pool) cudaEventDestroy(ev);
  for (int c = 0; c < 2; ++c) {
    if (g->sx[c]) cudaFree(g->sx[c]);
    if (g->sy[c]) cudaFree(g->sy[c]);
    if (g->sp_[c]) cudaFree(g->sp_[c]);
    if (g->hx[c]) cudaFreeHost(g->hx[c]);
    if (g->hy[c]) cudaFreeHost(g->hy[c]);
    if (g->hp[c]) cudaFreeHost(g->hp[c]);
    if (g->ev_h2d[c]) cudaEventDestroy(g->ev_h2d[c]);
    if (g->ev_used[c]) cudaEventDestroy(g->ev_used[c]);
    void *per[] = {g->pt2[c], g->ekey2[c], g->ka2[c], g->va2[c], g->kb2[c], g->vb2[c], g->item2[c], g->posrec2[c],
                   g->t2_2[c]};
    for (void *p : per)
      if (p) cudaFree(p);
    if (g->evF[c]) cudaEventDestroy(g->evF[c]);
    if (g->evB[c]) cudaEventDestroy(g->evB[c]);
  }
  if (g->cstream) cudaStreamDestroy(g->cstream);
  for (auto &ge : g->graphs) cudaGraphExecDestroy(ge.exec);
  if (g->capstream) cudaStreamDestroy(g->capstream);
  for (void *q : {(void *)g->gx, (void *)g->gy, (void *)g->gp})
    if (q) cudaFree(q);
  if (g->bstream) cudaStreamDestroy(g->bstream);
  delete g;
  return 0;
}

int fibar_set_stream(fibar_engine *g, void *stream) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  g->L.stream = (cudaStream_t)stream;
  return 0;
}

int fibar_reset(fibar_engine *g) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  return init_state(g);
}

int fibar_process(fibar_engine *g, const uint16_t *x, const uint16_t *y, const int8_t *p, int64_t n, int32_t mem) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  if (n <= 0) return 0;
  long long off = 0;
  if (mem == FIBAR_MEM_DEVICE) {
    // contiguous device packets are coalesced without copies: the batch reads
    // them in place (the caller keeps them alive until the next flush point)
    if (g->hfill > 0) {
      int rc = launch_host_batch(g);
      if (rc) return rc;
    }
    while (off < n) {
      if (g->zn > 0 && !(x + off == g->zx + g->zn && y + off == g->zy + g->zn && p + off == g->zp + g->zn)) {
        const long long zn = g->zn;
        g->zn = 0;
        int rc = run_batch_raw(g, g->zx, g->zy, g->zp, zn, nullptr);
        if (rc) return rc;
      }
      if (g->zn == 0) {
        g->zx = x + off;
        g->zy = y + off;
        g->zp = p + off;
      }
      const long long take = std::min((long long)n - off, g->Bcap - g->zn);
      g->zn += take;
      off += take;
      if (g->zn == g->Bcap) {
        const long long zn = g->zn;
        g->zn = 0;
        int rc = run_batch_raw(g, g->zx, g->zy, g->zp, zn, nullptr);
        if (rc) return rc;
      }
    }
    return 0;
  }
  if (g->zn > 0) {
    int rc = run_batch(g);
    if (rc) return rc;
  }
  // large packets already in pinned memory are DMA'd straight into the device
  // staging set (no CPU copy); the call returns once those copies are done,
  // so the caller may reuse its buffers as with any host packet
  const long long dmin = direct_min(g);
  const bool direct = n - off >= dmin && is_pinned(x) && is_pinned(y) && is_pinned(p);
  cudaEvent_t last_direct = nullptr;
  if (direct && g->hfill > 0) {   // earlier staged packets go first
    int rc = launch_host_batch(g);
    if (rc) return rc;
  }
  while (direct && n - off >= dmin) {
    const int c = g->cur;
    const long long take = std::min((long long)n - off, g->Bcap);
    CK(cudaStreamWaitEvent(g->cstream, g->ev_used[c], 0));
    CK(cudaMemcpyAsync(g->sx[c], x + off, sizeof(uint16_t) * take, cudaMemcpyHostToDevice, g->cstream));
    CK(cudaMemcpyAsync(g->sy[c], y + off, sizeof(uint16_t) * take, cudaMemcpyHostToDevice, g->cstream));
    CK(cudaMemcpyAsync(g->sp_[c], p + off, sizeof(int8_t) * take, cudaMemcpyHostToDevice, g->cstream));
    CK(cudaEventRecord(g->ev_h2d[c], g->cstream));
    CK(cudaStreamWaitEvent(g->L.stream, g->ev_h2d[c], 0));
    last_direct = g->ev_h2d[c];
    g->cur ^= 1;
    off += take;
    int rc = run_batch_raw(g, g->sx[c], g->sy[c], g->sp_[c], take, g->ev_used[c]);
    if (rc) return rc;
  }
  if (last_direct) CK(cudaEventSynchronize(last_direct));
  while (off < n) {
    if (g->hfill == 0) CK(cudaEventSynchronize(g->ev_h2d[g->cur]));   // host set free again
    const long long take = std::min((long long)n - off, g->Bcap - g->hfill);
    memcpy(g->hx[g->cur] + g->hfill, x + off, sizeof(uint16_t) * take);
    memcpy(g->hy[g->cur] + g->hfill, y + off, sizeof(uint16_t) * take);
    memcpy(g->hp[g->cur] + g->hfill, p + off, sizeof(int8_t) * take);
    g->hfill += take;
    off += take;
    if (g->hfill == g->Bcap) {
      int rc = launch_host_batch(g);
      if (rc) return rc;
    }
  }
  return 0;
}

int fibar_flush(fibar_engine *g) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  return sync_point(g);
}

int fibar_pending(fibar_engine *g, int64_t *device_events, int64_t *staged_events) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  if (device_events) *device_events = g->zn;
  if (staged_events) *staged_events = g->hfill;
  return 0;
}

int fibar_render(fibar_engine *g, int32_t mode, double fixed_bound, uint8_t *out, int32_t out_mem, double *bounds,
                 int32_t *degenerate) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  int rc = sync_point(g);
  if (rc) return rc;
  return render_core(g->L, g->l, g->n_pix, mode, fixed_bound, out, out_mem, bounds, degenerate, g->sel, g->frame, g->nsm);
}

int fibar_render_grid(const float *l_dev, int64_t n, int32_t mode, double fixed_bound, uint8_t *out, int32_t out_mem,
                      double *bounds, int32_t *degenerate, void *stream) {
  static SelState *sel = nullptr;
  static uint8_t *frame = nullptr;
  static long long cap = 0;
  static Launcher L;
  static int nsm = 0;
  if (!l_dev || n < 1) return fail(FIBAR_E_CONFIG, "empty grid");
  if (!sel) {
    int rc = dalloc(&sel, 1);
    if (rc) return rc;
    CK(cudaMemset(sel, 0, sizeof(SelState)));
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  if (out_mem != FIBAR_MEM_DEVICE && n > cap) {
    if (frame) cudaFree(frame);
    frame = nullptr;
    int rc = dalloc(&frame, n);
    if (rc) return rc;
    cap = n;
  }
  L.stream = (cudaStream_t)stream;
  return render_core(L, l_dev, n, mode, fixed_bound, out, out_mem, bounds, degenerate, sel, frame, nsm);
}

int fibar_read_qs(fibar_engine *g, int64_t qs[10]) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  int rc = sync_point(g);
  if (rc) return rc;
  DevState h;
  CK(cudaMemcpyAsync(&h, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, g->L.stream));
  CK(cudaStreamSynchronize(g->L.stream));
  qs[0] = h.s % (g->n_pix + 1);
  qs[1] = h.E - h.s;
  qs[2] = h.q;
  qs[3] = h.npix;
  qs[4] = h.ntiles;
  qs[5] = h.blur;
  qs[6] = h.stale;
  qs[7] = h.qtmin;
  qs[8] = h.qtmax;
  qs[9] = h.evctr;
  if (!g->spatial) {
    qs[0] = 0;
    qs[1] = 0;
  }
  return 0;
}

int fibar_counters(fibar_engine *g, int64_t *event_count, int64_t *oob_dropped) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  int rc = sync_point(g);
  if (rc) return rc;
  DevState h;
  CK(cudaMemcpyAsync(&h, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, g->L.stream));
  CK(cudaStreamSynchronize(g->L.stream));
  if (event_count) *event_count = h.E;
  if (oob_dropped) *oob_dropped = h.oob;
  return 0;
}

int fibar_read_state(fibar_engine *g, float *p_bar, float *l, uint16_t *active, uint8_t *tiles, uint16_t *qx,
                     uint16_t *qy) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  int rc = sync_point(g);
  if (rc) return rc;
  cudaStream_t s = g->L.stream;
  const long long n = g->n_pix;
  if (p_bar) CK(cudaMemcpyAsync(p_bar, g->pbar, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
  if (l) CK(cudaMemcpyAsync(l, g->l, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
  if (active || tiles || qx || qy) {
    if (!g->cnt_tmp) {
      rc |= dalloc(&g->cnt_tmp, n);
      rc |= dalloc(&g->tcnt_tmp, g->n_tiles);
      rc |= dalloc(&g->q_tmp, 2 * (n + 1));
      if (rc) return rc;
    }
    CK(cudaMemsetAsync(g->cnt_tmp, 0, sizeof(unsigned) * n, s));
    CK(cudaMemsetAsync(g->tcnt_tmp, 0, sizeof(unsigned) * g->n_tiles, s));
    Ctx x = g->ctx(nullptr, nullptr, 0, 0);
    if (g->spatial) {
      fibar_launch(g->L, "state_active", k_active_counts, g->nsm * 4, TPB, 0, s, x, g->cnt_tmp);
      fibar_launch(g->L, "state_tiles", k_tile_counts, g->nsm * 4, TPB, 0, s, x, g->cnt_tmp, g->tcnt_tmp);
      fibar_launch(g->L, "state_ring", k_ring_xy, g->nsm * 4, TPB, 0, s, x, g->q_tmp, g->q_tmp + n + 1);
    } else {
      CK(cudaMemsetAsync(g->q_tmp, 0, sizeof(uint16_t) * 2 * (n + 1), s));
    }
    CK(cudaGetLastError());
    std::vector<unsigned> hc, ht;
    if (active) hc.resize(n);
    if (tiles) ht.resize(g->n_tiles);
    if (active) CK(cudaMemcpyAsync(hc.data(), g->cnt_tmp, sizeof(unsigned) * n, cudaMemcpyDeviceToHost, s));
    if (tiles) CK(cudaMemcpyAsync(ht.data(), g->tcnt_tmp, sizeof(unsigned) * g->n_tiles, cudaMemcpyDeviceToHost, s));
    if (qx) CK(cudaMemcpyAsync(qx, g->q_tmp, sizeof(uint16_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    if (qy) CK(cudaMemcpyAsync(qy, g->q_tmp + n + 1, sizeof(uint16_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (active)
      for (long long i = 0; i < n; ++i) active[i] = (uint16_t)std::min<unsigned>(hc[i], 65535u);
    if (tiles)
      for (long long i = 0; i < g->n_tiles; ++i) tiles[i] = (uint8_t)std::min<unsigned>(ht[i], 255u);
  }
  CK(cudaStreamSynchronize(s));
  return 0;
}

int fibar_stats(fibar_engine *g, int64_t stats[16]) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  int rc = sync_point(g);
  if (rc) return rc;
  DevState h;
  CK(cudaMemcpyAsync(&h, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, g->L.stream));
  CK(cudaStreamSynchronize(g->L.stream));
  stats[0] = g->L.launches;
  stats[1] = g->batches;
  stats[2] = h.chunks;
  stats[3] = h.mismatch;
  stats[4] = h.pops;
  // tile_count (u8) can only saturate when a tile has more than 255 pixels
  stats[5] = h.saturated + ((g->spatial && g->A > 255 && h.E > 0) ? 1 : 0);
  stats[6] = h.E;
  stats[7] = g->Bcap;
  stats[8] = h.warm_pops;
  stats[9] = h.coop_iters;
  stats[10] = h.fix_rounds;
  stats[11] = h.dbg_bad;
  return 0;
}

int fibar_profile(fibar_engine *g, int32_t enable) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  join_blur(g);
  CK(cudaStreamSynchronize(g->L.stream));
  g->L.prof = enable != 0;
  g->L.recs.clear();
  g->L.used = 0;
  return 0;
}

int fibar_profile_read(fibar_engine *g, int32_t max_entries, char *names, int32_t name_len, double *total_ms,
                       int64_t *launches, int32_t *n_entries) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  join_blur(g);
  CK(cudaStreamSynchronize(g->L.stream));
  std::vector<std::string> keys;
  std::vector<double> ms;
  std::vector<long long> cnt;
  for (auto &r : g->L.recs) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, r.a, r.b));
    size_t k = 0;
    for (; k < keys.size(); ++k)
      if (keys[k] == r.name) break;
    if (k == keys.size()) {
      keys.push_back(r.name);
      ms.push_back(0.0);
      cnt.push_back(0);
    }
    ms[k] += t;
    cnt[k] += 1;
  }
  const int m = (int)std::min<size_t>(keys.size(), (size_t)max_entries);
  for (int k = 0; k < m; ++k) {
    strncpy(names + (size_t)k * name_len, keys[k].c_str(), name_len - 1);
    names[(size_t)k * name_len + name_len - 1] = 0;
    total_ms[k] = ms[k];
    launches[k] = cnt[k];
  }
  *n_entries = m;
  g->L.recs.clear();
  g->L.used = 0;
  return 0;
}

// debug: item completion / grab timestamps (ns) of the last batch; FIBAR_DEBUG_TIMES must be set
int fibar_debug_times(fibar_engine *g, uint64_t *done_ns, uint64_t *grab_ns, int64_t n) {
  if (!g || !g->dbg_t) return fail(FIBAR_E_CONFIG, "debug timestamps not enabled");
  join_blur(g);
  CK(cudaStreamSynchronize(g->L.stream));
  CK(cudaMemcpy(done_ns, g->dbg_t, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(grab_ns, g->dbg_g, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  return 0;
}

// debug: copy the blur prep records (80 B each) of the last batch
int fibar_debug_prep(fibar_engine *g, void *out, int64_t n) {
  if (!g || !g->prep) return fail(FIBAR_E_CONFIG, "no prep");
  join_blur(g);
  CK(cudaStreamSynchronize(g->L.stream));
  CK(cudaMemcpy(out, g->prep, sizeof(BlurPrep) * n, cudaMemcpyDeviceToHost));
  return 0;
}

int fibar_decode_evf1(const uint8_t *records, int64_t nrec, int32_t width, int32_t height, uint64_t t_base,
                      uint16_t *x, uint16_t *y, int8_t *p, uint64_t *t, int64_t *first_bad, void *stream) {
  if (nrec < 0 || !first_bad) return fail(FIBAR_E_CONFIG, "bad arguments");
  *first_bad = -1;
  if (nrec == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = (int)((nrec + EV_TILE - 1) / EV_TILE);
  unsigned *dt = nullptr;
  unsigned long long *bsum = nullptr, *bad = nullptr;
  CK(cudaMallocAsync((void **)&dt, sizeof(unsigned) * nrec, s));
  CK(cudaMallocAsync((void **)&bsum, sizeof(unsigned long long) * (nb + 1), s));
  CK(cudaMallocAsync((void **)&bad, sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), s));
  k_evf1_decode<<<nb, TPB, 0, s>>>(reinterpret_cast<const uint4 *>(records), reinterpret_cast<const uint2 *>(records),
                                   nrec, width, height, x, y, p, dt, bsum, bad);
  k_evf1_block_scan<<<1, 1024, 0, s>>>(bsum, nb, (unsigned long long)t_base);
  if (t) k_evf1_times<<<nb, TPB, 0, s>>>(dt, nrec, bsum, reinterpret_cast<unsigned long long *>(t));
  unsigned long long hb = 0;
  CK(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(dt, s);
  cudaFreeAsync(bsum, s);
  cudaFreeAsync(bad, s);
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  *first_bad = hb == ~0ull ? -1 : (int64_t)hb;
  return 0;
}

int fibar_copy_brightness(fibar_engine *g, float *dst, int32_t dst_mem) {
  if (!g || !dst) return fail(FIBAR_E_CONFIG, "null argument");
  int rc = sync_point(g);
  if (rc) return rc;
  CK(cudaMemcpyAsync(dst, g->l, sizeof(float) * g->n_pix,
                     dst_mem == FIBAR_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, g->L.stream));
  if (dst_mem != FIBAR_MEM_DEVICE) CK(cudaStreamSynchronize(g->L.stream));
  return 0;
}

int fibar_brightness_ptr(fibar_engine *g, float **out) {
  if (!g || !out) return fail(FIBAR_E_CONFIG, "null argument");
  int rc = sync_point(g);
  if (rc) return rc;
  *out = g->l;
  return 0;
}

}  // extern "C"
