// fibar_stage.cu -- per-pixel temporal replay (short and long segments), the blur
// dataflow (tap resolution + persistent polling grid) and the end-of-batch pass.
#include "fibar_kernels.cuh"

namespace fibar {

// -------------------------------------------------------------- temporal ---

// Per sorted position, fully parallel: the event's polarity gathered into
// sorted order and (filter ON) whether the event is evicted stale in this
// batch -- the random loads the serial per-pixel replay would otherwise wait on.
// the batch's counters into the engine state (k_batch_end, or the last block
// of the front end's final k_posinfo)
__device__ __forceinline__ void close_batch(const Ctx &x) {
  DevState *s = x.st;
  const BatchState *bsp = x.bs;
  s->E += bsp->B;
  if (x.spatial) {
    s->stale += bsp->stale_batch;
    if (x.blur_on) s->blur += bsp->stale_batch;
  }
}

// close != 0: the last block to finish also closes the batch (saves a launch
// on the front end's critical chain)
__global__ void __launch_bounds__(TPB) k_posinfo(Ctx x, int close) {
  pdl_wait();
  const long long B = x.bs->B;
  const long long i = (long long)blockIdx.x * TPB + threadIdx.x;
  if (i < B) {
    const unsigned jj = x.sidx[i];
    x.spol[i] = x.epol[jj];
    if (x.spatial) {
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
  }
  if (close) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&x.bs->nclosed, 1u) == gridDim.x - 1) {
        __threadfence();
        close_batch(x);
      }
    }
  }
}

// One thread per pixel segment replays its events in stream order with the
// reference's float32 operation order (_kernels.py:67-73 / 124-130).  Inputs
// are read GROUP positions at a time (all loads issued before the dependent
// arithmetic), so long segments (hot pixels) run at the arithmetic chain's speed.

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
    if (slot < x.max_long) x.longseg[slot] = make_uint2((unsigned)i, c);
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
  if (end - i > LONG_SEG) return;   // long segment (hot pixel): k_temporal_long (listed by k_link), beside this kernel
  unsigned carry = prc.carried;
  if (carry != FIBAR_NONE) x.item[carry].runpos = (unsigned)i;
  float pb = x.pbar[c], lv = x.l[c];
  const float g = x.use_gain ? x.gain[c] : 1.0f;
  // inputs in groups of RGROUP positions, the next group's loads in flight
  // while this group's chain runs (a segment of hundreds of events runs at
  // the arithmetic chain's speed, not one L2 round trip per group)
  constexpr int RGROUP = 16;
  int8_t pa[RGROUP], pbuf[RGROUP];
  unsigned ba[RGROUP], bbuf[RGROUP];
  auto load = [&](long long q0, int8_t (&pol)[RGROUP], unsigned (&bi)[RGROUP]) {
#pragma unroll
    for (int u = 0; u < RGROUP; ++u) {
      const long long q = q0 + u;
      pol[u] = q < end ? x.spol[q] : (int8_t)0;
      bi[u] = q < end ? x.posrec[q].bidx : FIBAR_NONE;
    }
  };
  auto step = [&](long long q0, const int8_t (&pol)[RGROUP], const unsigned (&bi)[RGROUP]) {
#pragma unroll
    for (int u = 0; u < RGROUP; ++u) {
      const long long q = q0 + u;
      if (q >= end) break;
      const float p = (float)pol[u];
      pb = faddr(fmulr(x.alpha, pb), fmulr(x.oma, p));
      float d = fsubr(p, pb);
      if (x.use_gain) d = fmulr(d, g);
      const float tt = fmulr(x.h, d);
      lv = faddr(fmulr(x.beta, lv), tt);
      x.t2[q] = tt;
      *reinterpret_cast<uint2 *>(&x.posrec[q].runbase) = make_uint2(carry, __float_as_uint(lv));
      if (bi[u] != FIBAR_NONE) {
        carry = bi[u];
        if (q + 1 < end) x.item[bi[u]].runpos = (unsigned)(q + 1);
      }
    }
  };
  if (end - i <= 4) {   // the common short segment: no group machinery
#pragma unroll 1
    for (long long q = i; q < end; ++q) {
      const float p = (float)x.spol[q];
      const unsigned bq = x.posrec[q].bidx;
      pb = faddr(fmulr(x.alpha, pb), fmulr(x.oma, p));
      float d = fsubr(p, pb);
      if (x.use_gain) d = fmulr(d, g);
      const float tt = fmulr(x.h, d);
      lv = faddr(fmulr(x.beta, lv), tt);
      x.t2[q] = tt;
      *reinterpret_cast<uint2 *>(&x.posrec[q].runbase) = make_uint2(carry, __float_as_uint(lv));
      if (bq != FIBAR_NONE) {
        carry = bq;
        if (q + 1 < end) x.item[bq].runpos = (unsigned)(q + 1);
      }
    }
  } else {
    long long pos = i;
    load(pos, pa, ba);
    while (pos < end) {
      const long long nx = pos + RGROUP;
      if (nx < end) load(nx, pbuf, bbuf);
      step(pos, pa, ba);
      if (nx >= end) break;
      const long long nn = nx + RGROUP;
      if (nn < end) load(nn, pa, ba);
      step(nx, pbuf, bbuf);
      pos = nn;
    }
  }
  x.pbar[c] = pb;
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
// loaded PGROUP at a time with the next group's loads in flight while this
// group's chain runs
__device__ __forceinline__ void replay_piece(const Ctx &x, long long q0, long long q1, float &pb, float &lv, float g,
                                             bool write) {
  constexpr int PGROUP = 16;
  int8_t pa[PGROUP], pbuf[PGROUP];
  auto load = [&](long long s0, int8_t (&pol)[PGROUP]) {
#pragma unroll
    for (int u = 0; u < PGROUP; ++u) pol[u] = s0 + u < q1 ? x.spol[s0 + u] : (int8_t)0;
  };
  auto step = [&](long long s0, const int8_t (&pol)[PGROUP]) {
#pragma unroll
    for (int u = 0; u < PGROUP; ++u) {
      if (s0 + u >= q1) break;
      float tt;
      iir_step(x, pb, lv, (float)pol[u], g, tt);
      if (write && x.spatial) {
        x.t2[s0 + u] = tt;
        x.posrec[s0 + u].val = lv;
      }
    }
  };
  long long q = q0;
  if (q < q1) load(q, pa);
  while (q < q1) {
    const long long nx = q + PGROUP;
    if (nx < q1) load(nx, pbuf);
    step(q, pa);
    if (nx >= q1) break;
    const long long nn = nx + PGROUP;
    if (nn < q1) load(nn, pa);
    step(nx, pbuf);
    q = nn;
  }
}


// One IIR step on polarity p from shared memory; WRITE: the per-position outputs
template <bool WRITE>
__device__ __forceinline__ void iir_step_s(const Ctx &x, float &pb, float &lv, int pol, float g, long long q) {
  float tt;
  iir_step(x, pb, lv, (float)pol, g, tt);
  if (WRITE) {
    x.t2[q] = tt;
    x.posrec[q].val = lv;
  }
}

// replay the staged polarities sp[i0, i1) (global positions gq + i) from (pb, lv)
template <bool WRITE>
__device__ __forceinline__ void replay_smem(const Ctx &x, const int8_t *sp, int i0, int i1, float &pb, float &lv,
                                            float g, long long gq) {
  int i = i0;
  for (; i < i1 && (i & 3); ++i) iir_step_s<WRITE>(x, pb, lv, sp[i], g, gq + i);
#pragma unroll 2
  for (; i + 4 <= i1; i += 4) {
    const int w = *reinterpret_cast<const int *>(sp + i);
    iir_step_s<WRITE>(x, pb, lv, (int)(int8_t)(w & 0xFF), g, gq + i);
    iir_step_s<WRITE>(x, pb, lv, (int)(int8_t)((w >> 8) & 0xFF), g, gq + i + 1);
    iir_step_s<WRITE>(x, pb, lv, (int)(int8_t)((w >> 16) & 0xFF), g, gq + i + 2);
    iir_step_s<WRITE>(x, pb, lv, (int)(w >> 24), g, gq + i + 3);
  }
  for (; i < i1; ++i) iir_step_s<WRITE>(x, pb, lv, sp[i], g, gq + i);
}

constexpr int LT_TILE = 8192;            // events of a segment staged in shared memory at a time
constexpr int LT_PMIN = 8;               // fewest events per lane
constexpr long long LT_BIG = 1 << 17;    // longer segments: pieces of thousands of events straight from global memory

__global__ void __launch_bounds__(LONG_TPB) k_temporal_long(Ctx x) {
  pdl_wait();
  __shared__ float s_spb[LONG_TPB], s_slv[LONG_TPB], s_epb[LONG_TPB], s_elv[LONG_TPB];
  __shared__ unsigned s_last[LONG_TPB];
  __shared__ __align__(16) int8_t s_pol[LT_TILE];
  __shared__ unsigned s_bidx[LT_TILE];
  __shared__ unsigned s_wlast[LONG_TPB / 32];
  __shared__ int s_bad;
  const unsigned n = min(x.bs->nlong, x.max_long);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
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
    const float g = x.use_gain ? x.gain[c] : 1.0f;
    const long long len = end - st;
    if (len <= LT_BIG) {
      // Tiles of the segment staged in shared memory (polarities and, filter
      // ON, which blur each position carries).  Lane i takes the i-th piece of
      // the tile: it starts twarm events early from zero (the float32
      // recurrences contract, see above), or from the tile's exact start state
      // when that is no further away, and every piece's start is checked
      // against its left neighbour's end.
      float pb0 = x.pbar[c], lv0 = x.l[c];
      unsigned carry0 = x.spatial ? x.pt[c].carried : FIBAR_NONE;
      if (x.spatial && tid == 0 && carry0 != FIBAR_NONE) x.item[carry0].runpos = (unsigned)st;
      for (long long t0 = st; t0 < end; t0 += LT_TILE) {
        const int tlen = (int)min((long long)LT_TILE, end - t0);
        {
          // staging: 16-byte loads over the aligned middle, bytes at the ends
          const long long a0 = (t0 + 15) & ~15LL, a1 = (t0 + tlen) & ~15LL;
          if (a0 < a1) {
            for (long long q = a0 + 16LL * tid; q < a1; q += 16LL * LONG_TPB) {
              const int4 v = *reinterpret_cast<const int4 *>(x.spol + q);
              const int o = (int)(q - t0);
              int8_t *d = s_pol + o;
              if ((o & 15) == 0) {
                *reinterpret_cast<int4 *>(d) = v;
              } else {
                const int w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int b = 0; b < 16; ++b) d[b] = (int8_t)(w[b >> 2] >> (8 * (b & 3)));
              }
            }
            for (long long q = t0 + tid; q < a0; q += LONG_TPB) s_pol[q - t0] = x.spol[q];
            for (long long q = a1 + tid; q < t0 + tlen; q += LONG_TPB) s_pol[q - t0] = x.spol[q];
          } else {
            for (int i = tid; i < tlen; i += LONG_TPB) s_pol[i] = x.spol[t0 + i];
          }
          if (x.spatial)
            for (int i = tid; i < tlen; i += LONG_TPB) s_bidx[i] = x.posrec[t0 + i].bidx;
        }
        __syncthreads();
        const int P = max(LT_PMIN, (tlen + LONG_TPB - 1) / LONG_TPB);
        const int lanes = (tlen + P - 1) / P;
        const bool on = tid < lanes;
        const int q0 = on ? tid * P : tlen, q1 = on ? min(tlen, q0 + P) : tlen;
        float pb = 0.0f, lv = 0.0f;
        if (on) {
          if (q0 <= x.twarm) {
            pb = pb0;
            lv = lv0;
            replay_smem<false>(x, s_pol, 0, q0, pb, lv, g, t0);
          } else {
            replay_smem<false>(x, s_pol, q0 - x.twarm, q0, pb, lv, g, t0);
          }
        }
        s_spb[tid] = pb;   // (speculative) state at the piece start
        s_slv[tid] = lv;
        if (x.spatial) replay_smem<true>(x, s_pol, q0, q1, pb, lv, g, t0);
        else replay_smem<false>(x, s_pol, q0, q1, pb, lv, g, t0);
        s_epb[tid] = pb;
        s_elv[tid] = lv;
        if (tid == 0) s_bad = 0;
        __syncthreads();
        if (on && tid > 0 && (__float_as_uint(s_spb[tid]) != __float_as_uint(s_epb[tid - 1]) ||
                              __float_as_uint(s_slv[tid]) != __float_as_uint(s_elv[tid - 1])))
          atomicMax(&s_bad, 1);
        __syncthreads();
        if (s_bad) {
          // rare: re-run the pieces whose start was wrong, in lane order, from the exact states
          for (int i = 1; i < lanes; ++i) {
            if (tid == i && (__float_as_uint(s_spb[i]) != __float_as_uint(s_epb[i - 1]) ||
                             __float_as_uint(s_slv[i]) != __float_as_uint(s_elv[i - 1]))) {
              pb = s_epb[i - 1];
              lv = s_elv[i - 1];
              s_spb[i] = pb;
              s_slv[i] = lv;
              if (x.spatial) replay_smem<true>(x, s_pol, q0, q1, pb, lv, g, t0);
              else replay_smem<false>(x, s_pol, q0, q1, pb, lv, g, t0);
              s_epb[i] = pb;
              s_elv[i] = lv;
            }
            __syncthreads();
          }
        }
        pb0 = s_epb[lanes - 1];
        lv0 = s_elv[lanes - 1];
        if (x.spatial) {
          // which blur each position builds on: the last stale event before it
          // in the segment, or the pixel's carried blur
          unsigned last = FIBAR_NONE;
          for (int i = q0; i < q1; ++i)
            if (s_bidx[i] != FIBAR_NONE) last = s_bidx[i];
          const unsigned m = __ballot_sync(0xffffffffu, last != FIBAR_NONE);
          if (lane == 31 - __clz(m | 1u) || (m == 0 && lane == 0)) s_wlast[wid] = m ? last : FIBAR_NONE;
          __syncthreads();
          unsigned carry = FIBAR_NONE;
          const unsigned below = m & ((1u << lane) - 1u);
          const unsigned from_lane = __shfl_sync(0xffffffffu, last, below ? 31 - __clz(below) : 0);
          if (below) {
            carry = from_lane;
          } else {
            for (int w = wid - 1; w >= 0; --w)
              if (s_wlast[w] != FIBAR_NONE) {
                carry = s_wlast[w];
                break;
              }
            if (carry == FIBAR_NONE) carry = carry0;
          }
          for (int i = q0; i < q1; ++i) {
            x.posrec[t0 + i].runbase = carry;
            const unsigned bi = s_bidx[i];
            if (bi != FIBAR_NONE) {
              carry = bi;
              if (t0 + i + 1 < end) x.item[bi].runpos = (unsigned)(t0 + i + 1);
            }
          }
          for (int w = LONG_TPB / 32 - 1; w >= 0; --w)
            if (s_wlast[w] != FIBAR_NONE) {
              carry0 = s_wlast[w];
              break;
            }
        }
        __syncthreads();   // the tile's shared arrays are rewritten next
      }
      if (tid == 0) {
        x.pbar[c] = pb0;
        if (!x.spatial) x.l[c] = lv0;
      }
      continue;
    }
    const int lanes = (int)min((long long)LONG_TPB, max(32LL, len / LONG_PIECE));
    const long long P = (len + lanes - 1) / lanes;
    const bool on = tid < lanes;
    const long long q0 = on ? min(end, st + tid * P) : end, q1 = on ? min(end, q0 + P) : end;
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
    if (tid == 0) x.pbar[c] = fpb;
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



// First resolution of item p's 3x3 taps (_kernels.py:174-188 tap order).  A
// tap's brightness "at item p" is the neighbour's value after every temporal
// update up to the popping event and every earlier blur.  It comes from the
// pixel record (batch segment, carried blur) and the position record of the
// neighbour's latest event at that time: directly (batch-start value or
// first-run value) or, when a blur produced it, after that blur's flag.
// Runs for all items in parallel, before any blur (no waiting).
__device__ __forceinline__ void prep_item(const Ctx &x, unsigned p);

// Stale items are visited in pixel (tile-major sorted) order, not pop order:
// a sorted position whose event is evicted stale names its item, a segment
// head names its pixel's carried item, and k_popj lists the carried items of
// pixels without events.  Neighbouring threads then resolve neighbouring
// pixels' 3x3 taps, so the random pixel / position records they read are
// shared in L1 instead of fetched again from L2.
__global__ void __launch_bounds__(TPB, PREP_MINB) k_blur_prep(Ctx x) {
  pdl_wait();
  const long long B = x.bs->B;
  const long long q = (long long)blockIdx.x * TPB + threadIdx.x;
  if (q < B) {
    const unsigned bidx = x.posrec[q].bidx;
    if (bidx != FIBAR_NONE) prep_item(x, bidx);
    if (q == 0 || x.skey[q - 1] != x.skey[q]) {
      const unsigned carried = x.pt[x.ekey[x.sidx[q]]].carried;
      if (carried != FIBAR_NONE) prep_item(x, carried);
    }
  } else {
    // the threads past the batch's events (at least nsm blocks of them) stride
    // over the carried-only list, up to one entry per eviction
    const long long nco = (long long)x.bs->nco, tail = (long long)gridDim.x * TPB - B;
    for (long long k = q - B; k < nco; k += tail) prep_item(x, x.colist[k]);
  }
}

__device__ __forceinline__ void prep_item(const Ctx &x, unsigned p) {
  const Item it = x.item[p];
  BlurPrep out;
  out.okm = 0;
  out.pend = 0;
  const unsigned jrel = it.jrel;
  const int cx = (int)(it.pix % (unsigned)x.W), cy = (int)(it.pix / (unsigned)x.W);
  if (x.halo) {
    // halo band: items outside the band's rows are not this engine's; the
    // outermost halo rows take their blurred values from the neighbours
    if (cy < x.hreg0 || cy >= x.hreg1) {
      x.prep[p].okm = 0;
      return;
    }
    if (cy == x.hin_top || cy == x.hin_bot) {
      out.okm = HALO_OKM;
      out.val[0] = x.hslot[p];
      out.runpos = it.runpos;
      x.prep[p] = out;
      return;
    }
  }
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
                                                float v, unsigned hi) {
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
      st_relaxed_u64(&x.mv64[r + u], ((unsigned long long)hi << 32) | __float_as_uint(v));
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
template <bool HALO>
__device__ __forceinline__ void blur_lanes(const Ctx &x) {
  pdl_wait();
  const BatchScalars b = load_bs(x);
  const unsigned npop = (unsigned)(b.s_end - b.s_start);
  const int lane = threadIdx.x & 31;
  unsigned p = FIBAR_NONE, okm = 0, pend = 0, runpos = FIBAR_NONE;
  unsigned tnt = 0;   // halo bands: the value read a not-yet-final halo value (TAINT_HI or 0)
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
          tnt = 0;
          if (okm && HALO && b.epoch != b.epoch0) {
            // a later exchange round: an item already final (untainted) in an
            // earlier round of this batch keeps its value and its rebuilt run
            const unsigned hw = (unsigned)(ld_relaxed_u64(&x.bv64[q]) >> 32);
            if (!(hw & TAINT_HI) && hw >= b.epoch0) okm = 0;
          }
          if (HALO && okm == HALO_OKM) {
            // injected halo item: its blurred value comes from the neighbour
            const unsigned long long w = x.hin[n0.z];
            p = q;
            pend = 0;
            val[0] = (unsigned)w;
            tnt = (unsigned)(w >> 32) & TAINT_HI;
            runpos = __ldcg(rec + 2).w;
          } else if (okm) {
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
            if (x.dbg_g) {
              unsigned long long tt;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
              x.dbg_g[q] = tt;
            }
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
        const unsigned hw = (unsigned)(w >> 32);
        if (hw != b.epoch) {
          // halo bands: this round's word (tainted) or a final one from an
          // earlier round of the batch; otherwise not there yet
          const unsigned e = hw & ~TAINT_HI;
          if (!(HALO && e >= b.epoch0 && (e == b.epoch || !(hw & TAINT_HI)))) continue;
          tnt |= hw & TAINT_HI;
        }
        val[t] = (unsigned)w;
        pend &= ~(1u << t);
      }
      if (pend == 0) {
        float v;
        if (HALO && okm == HALO_OKM) {
          v = __uint_as_float(val[0]);
        } else {
          float num = 0.0f, den = 0.0f;
#pragma unroll
          for (int t = 0; t < 9; ++t) {
            if (!((okm >> t) & 1)) continue;
            const float w = (float)((t / 3 == 1 ? 2 : 1) * (t % 3 == 1 ? 2 : 1));
            num = faddr(num, fmulr(w, __uint_as_float(val[t])));
            den = faddr(den, w);
          }
          v = __fdiv_rn(num, den);
        }
        const unsigned hi = b.epoch | tnt;
        st_relaxed_u64(&x.bv64[p], ((unsigned long long)hi << 32) | __float_as_uint(v));
        if (x.dbg_t) {
          unsigned long long tt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
          x.dbg_t[p] = tt;
        }
        if (runpos != FIBAR_NONE) materialise_run(x, b, p, runpos, v, hi);
        p = FIBAR_NONE;
      } else if (x.blur_sleep) {
        __nanosleep(x.blur_sleep);
      }
    }
    if (__all_sync(0xffffffffu, exhausted && p == FIBAR_NONE)) break;
  }
}

__global__ void __launch_bounds__(TPB, BLUR_MINB) k_blur(Ctx x) { blur_lanes<false>(x); }
__global__ void __launch_bounds__(TPB) k_blur_halo(Ctx x) { blur_lanes<true>(x); }

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

// ------------------------------------------------------------ halo band ---
// Filter-ON row bands.  Each rank blurs the items of its rows
// plus a halo of G rows; the outermost halo row's items are injected from the
// neighbour that owns them.  The item lists are built from the global window
// (identical on every rank) in pop order, so both sides of a boundary agree
// on the order of the words they exchange without sending indices.

__device__ __forceinline__ unsigned halo_classes(const Ctx &x, unsigned p, unsigned npop) {
  if (p >= npop) return 0u;
  const unsigned pix = x.item[p].pix;
  if (pix == FIBAR_NONE) return 0u;
  const int row = (int)(pix / (unsigned)x.W);
  return (unsigned)(row == x.hin_top) | (unsigned)(row == x.hin_bot) << 1 | (unsigned)(row == x.hout_top) << 2 |
         (unsigned)(row == x.hout_bot) << 3;
}

// per block and class (in_top, in_bot, out_top, out_bot): item counts, laid
// out class-major so one exclusive scan gives every item its slot in the
// concatenated list [in_top | in_bot | out_top | out_bot]
__global__ void __launch_bounds__(TPB) k_halo_count(Ctx x, unsigned *cnt, int nb) {
  pdl_wait();
  const unsigned npop = (unsigned)x.bs->npop;
  const unsigned p = blockIdx.x * TPB + threadIdx.x;
  const unsigned cls = halo_classes(x, p, npop);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int n = __syncthreads_count((cls >> c) & 1u);
    if (threadIdx.x == 0) cnt[c * nb + blockIdx.x] = (unsigned)n;
  }
}

__global__ void __launch_bounds__(TPB) k_halo_write(Ctx x, const unsigned *cnt, int nb, unsigned *hlist) {
  pdl_wait();
  __shared__ unsigned wc[4][TPB / 32];
  const unsigned npop = (unsigned)x.bs->npop;
  const unsigned p = blockIdx.x * TPB + threadIdx.x;
  const unsigned cls = halo_classes(x, p, npop);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned below[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const unsigned m = __ballot_sync(0xffffffffu, (cls >> c) & 1u);
    below[c] = __popc(m & ((1u << lane) - 1u));
    if (lane == 0) wc[c][wid] = __popc(m);
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (!((cls >> c) & 1u)) continue;
    unsigned pos = cnt[c * nb + blockIdx.x] + below[c];
    for (int w = 0; w < wid; ++w) pos += wc[c][w];
    hlist[pos] = p;
    if (c < 2) x.hslot[p] = pos;   // in-words are [in_top | in_bot], the list's first part
  }
}

// next exchange round of the batch: a fresh epoch (this round's words) and ticket
__global__ void k_halo_epoch(Ctx x) {
  pdl_wait();
  x.st->epoch += 1;
  x.bs->epoch = x.st->epoch;
  x.bs->ticket = 0;
}

// out-words of the round: taint bit | float bits of the items the neighbours inject
__global__ void __launch_bounds__(TPB) k_halo_collect(Ctx x, const unsigned *hlist, long long n_in, long long n_out,
                                                      unsigned long long *out) {
  pdl_wait();
  const long long i = (long long)blockIdx.x * TPB + threadIdx.x;
  if (i >= n_out) return;
  const unsigned long long w = ld_relaxed_u64(&x.bv64[hlist[n_in + i]]);
  out[i] = (w & (1ull << 63)) | (w & 0xFFFFFFFFull);
}

__global__ void k_batch_end(Ctx x) {
  pdl_wait();
  close_batch(x);
}


}  // namespace fibar
