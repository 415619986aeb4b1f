// fibar_readout.cu -- read-out (exact percentile select + float64 map), EVF1 decode,
// state export and state initialisation kernels.
#include "fibar_kernels.cuh"

namespace fibar {

// ---------------------------------------------------------------- read-out ---


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
  // only the distinct targets' histograms are used (pass 0: one; later
  // passes: usually two), so only those are cleared, merged and read back
#pragma unroll
  for (int t = 0; t < 4; ++t)
    if (act[t])
      for (int i = threadIdx.x; i < 2048; i += TPB) h[t][i] = 0;
  __syncthreads();
  // brightness values cluster in a few top digits, so equal digits within a
  // warp are combined first (one shared atomic per distinct digit and target)
  const long long stride = (long long)gridDim.x * TPB;
  const long long n_round = (n + 31) & ~31LL;
  // SEL_UNROLL values per thread are loaded before any is binned, so a
  // thread waits on one memory round trip per SEL_UNROLL values
  constexpr int SEL_UNROLL = 8;
  for (long long i0 = (long long)blockIdx.x * TPB + threadIdx.x; i0 < n_round; i0 += SEL_UNROLL * stride) {
    unsigned kk[SEL_UNROLL];
#pragma unroll
    for (int u = 0; u < SEL_UNROLL; ++u) {
      const long long i = i0 + u * stride;
      kk[u] = i < n ? order_key(__ldg(&l[i])) : 0u;
    }
#pragma unroll
    for (int u = 0; u < SEL_UNROLL; ++u) {
      const long long i = i0 + u * stride;
      if (i >= n_round) break;   // warp-uniform (n_round and stride are multiples of 32)
      const bool in = i < n;
      const unsigned k = kk[u];
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
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    if (!act[t]) continue;
    for (int i = threadIdx.x; i < 2048; i += TPB) {
      const unsigned v = h[t][i];
      if (v) atomicAdd(&sel->hist[t][i], v);
    }
  }
  __threadfence();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(&sel->done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // totals into shared memory (and the global table cleared for the next pass)
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    if (!act[t]) continue;
    for (int i = threadIdx.x; i < 2048; i += TPB) {
      h[t][i] = __ldcg(&sel->hist[t][i]);
      sel->hist[t][i] = 0u;
    }
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


}  // namespace fibar
