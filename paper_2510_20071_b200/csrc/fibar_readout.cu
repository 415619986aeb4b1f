// fibar_readout.cu -- read-out (exact percentile select + float64 map), EVF1 decode,
// state export and state initialisation kernels.
#include "fibar_kernels.cuh"

namespace fibar {

// ---------------------------------------------------------------- read-out ---
//
// render() (pipeline.py:247-269): robust bounds are numpy's 'linear'
// percentiles 1 and 99 of l -- order statistics at ranks floor((n-1)q) and
// floor((n-1)q)+1 blended by _lerp -- then the float64 u8 map.  One cooperative
// kernel does all of it: each CTA (one per SM) reads its contiguous slice of l
// once (16-byte loads) into shared memory as order keys, and the grid selects
// the four order statistics exactly with a 3-pass MSB radix select (digits
// 11/11/10 bits).  Per pass every CTA histograms its keys in shared memory
// (warp-aggregated atomics) and adds the non-zero bins to a global histogram;
// the last CTA to arrive picks the digits from the totals and releases the
// others with them (a grid barrier).  After the last pass each CTA maps its own
// slice to u8.
// l is read from HBM/L2 once; the passes and the map run on chip.

// u8 = clip(floor((v - lo) * (255 / (hi - lo)) + 0.5), 0, 255) in float64
// (pipeline.py:265-268); degenerate grids render mid-gray (pipeline.py:260-263)
// FIBAR_RO_TIMES builds: CTA 0 records globaltimer stamps of its phases
#ifdef FIBAR_RO_TIMES
#define RO_TS(k)                                                                    \
  do {                                                                              \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                      \
      unsigned long long _t;                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                       \
      sel->ts[k] = _t;                                                              \
    }                                                                               \
  } while (0)
#else
#define RO_TS(k) \
  do {           \
  } while (0)
#endif

__device__ __forceinline__ unsigned ro_map(float v, double lo, double scale, bool deg) {
  if (deg) return 128u;
  const double s = __dmul_rn(__dsub_rn((double)v, lo), scale);
  double r = floor(__dadd_rn(s, 0.5));
  r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
  return (unsigned)r;
}

// Grid barrier with a serial step: every CTA arrives (release); the last one
// to arrive runs `last` (which reads what the others published and fills
// sel->bc) and releases the others, which then read sel->bc into s_bc.
// gen0 = the barrier generation read at kernel start; k = 1, 2, ...
template <class F>
__device__ __forceinline__ void ro_barrier(SelState *sel, unsigned gen0, unsigned k, unsigned *s_bc, bool *s_last,
                                           F &&last) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(&sel->bar_count) : "memory");
    *s_last = old == gridDim.x - 1;
  }
  __syncthreads();
  if (*s_last) {
    fence_acquire_gpu();
    last();
    __syncthreads();
    if (threadIdx.x == 0) {
      sel->bar_count = 0;
      __threadfence();
      st_release_u32(&sel->bar_gen, gen0 + k);
    }
  } else if (threadIdx.x == 0) {
    while (ld_acquire_u32(&sel->bar_gen) != gen0 + k) {
    }
  }
  if (threadIdx.x == 0) {   // every CTA (the last one too) reads what was published
    uint4 a, b, c;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(&sel->bc[0]) : "memory");
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(&sel->bc[4]) : "memory");
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "l"(&sel->bc[8]) : "memory");
    s_bc[0] = a.x; s_bc[1] = a.y; s_bc[2] = a.z; s_bc[3] = a.w;
    s_bc[4] = b.x; s_bc[5] = b.y; s_bc[6] = b.z; s_bc[7] = b.w;
    s_bc[8] = c.x; s_bc[9] = c.y; s_bc[10] = c.z; s_bc[11] = c.w;
  }
  __syncthreads();
}

#ifndef FIBAR_RO_MINB
#define FIBAR_RO_MINB 2
#endif
__global__ void __launch_bounds__(RO_TPB, FIBAR_RO_MINB)
    k_readout(const float *__restrict__ l, long long n, SelState *sel, int mode, double fixed_bound, uint4 ranks,
              double g_lo, double g_hi, uint8_t *__restrict__ out, long long slice, int on_chip) {
  extern __shared__ __align__(16) unsigned ro_keys[];
  __shared__ unsigned h[4][2048];
  __shared__ unsigned s_pref[4], s_rank[4], s_bc[12];
  constexpr unsigned RO_CL = 1024;
  __shared__ unsigned s_cl[RO_CL], s_ncl;
  __shared__ uint4 s_wt[RO_TPB / 32];
  __shared__ unsigned s_gen;
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  RO_TS(1);
  const long long beg = (long long)blockIdx.x * slice;
  const int cnt = (int)max(0LL, min(n, beg + slice) - beg);
  const bool robust = mode == FIBAR_RENDER_ROBUST;
  // a robust launch uses the counters of set sel->cur[par] and clears the
  // other set for the next one (fixed mode touches neither, nor the parity)
  const unsigned par = robust ? sel->parity : 0u;
  if (robust) {
    unsigned *other = reinterpret_cast<unsigned *>(&sel->cur[par ^ 1u]);
    constexpr int TOT = sizeof(SelCounters) / 4;
    for (int i = blockIdx.x * RO_TPB + tid; i < TOT; i += gridDim.x * RO_TPB) other[i] = 0u;
    if (tid == 0) s_gen = ld_acquire_u32(&sel->bar_gen);   // constant until this launch's first barrier
  }
  SelCounters &sc = sel->cur[par];
  const bool vec = on_chip && ((reinterpret_cast<unsigned long long>(l + beg) & 15ull) == 0);
  double lo, hi;
  if (robust) {
    if (on_chip) {
      if (vec) {
        const float4 *l4 = reinterpret_cast<const float4 *>(l + beg);
        for (int i = tid; i < (cnt >> 2); i += RO_TPB) {
          const float4 v = __ldcg(&l4[i]);
          reinterpret_cast<uint4 *>(ro_keys)[i] = make_uint4(order_key(v.x), order_key(v.y), order_key(v.z), order_key(v.w));
        }
        for (int i = (cnt & ~3) + tid; i < cnt; i += RO_TPB) ro_keys[i] = order_key(__ldcg(&l[beg + i]));
      } else {
        for (int i = tid; i < cnt; i += RO_TPB) ro_keys[i] = order_key(__ldcg(&l[beg + i]));
      }
    }
    if (tid == 0) s_ncl = 0u;
    if (tid < 4) {
      s_pref[tid] = 0u;
      s_rank[tid] = tid == 0 ? ranks.x : (tid == 1 ? ranks.y : (tid == 2 ? ranks.z : ranks.w));
    }
    __syncthreads();
    RO_TS(2);
    const unsigned gen0 = s_gen;
    unsigned nbar = 0;
    // ---- exact radix select (digits 11/11/10 bits, MSB first)
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
      const int shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
      const unsigned dmask = pass == 2 ? 1023u : 2047u;
      const unsigned hmask = pass == 0 ? 0u : (pass == 1 ? 0xFFE00000u : 0xFFFFFC00u);
      unsigned pref[4], rank[4];
      int src[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        pref[t] = s_pref[t];
        rank[t] = s_rank[t];   // read before the pass's first barrier; written after its last
        src[t] = t;
#pragma unroll
        for (int u = 0; u < t; ++u)
          if (src[t] == t && pref[u] == pref[t]) src[t] = u;
      }
      // pass 0: one histogram (every target's prefix is empty), counted into
      // four sub-histograms (warp w adds into h[w & 3]) to spread the
      // contention of clustered values, then summed into h[0]; passes 1-2:
      // one histogram per distinct prefix, few keys match
      const bool p0 = pass == 0;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (p0 || src[t] == t)
          for (int i = tid; i < 2048; i += RO_TPB) h[t][i] = 0u;
      __syncthreads();
      if (p0) {
        unsigned *hw = h[wid & 3];
        for (int i = tid; i < cnt; i += RO_TPB) {
          const unsigned k = on_chip ? ro_keys[i] : order_key(__ldcg(&l[beg + i]));
          atomicAdd(&hw[k >> 21], 1u);
        }
        __syncthreads();
        for (int i = tid; i < 2048; i += RO_TPB) h[0][i] += h[1][i] + h[2][i] + h[3][i];
      } else {
        // pass 1 scans the slice and keeps the keys matching a prefix (few) in
        // s_cl; pass 2 scans only those, unless they overflowed
        const bool from_list = pass == 2 && s_ncl <= RO_CL;
        const int nscan = from_list ? (int)s_ncl : cnt;
        for (int i = tid; i < nscan; i += RO_TPB) {
          const unsigned k = from_list ? s_cl[i] : (on_chip ? ro_keys[i] : order_key(__ldcg(&l[beg + i])));
          const unsigned d = (k >> shift) & dmask;
          bool any = false;
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if ((k & hmask) == pref[t]) {
              any = true;
              if (src[t] == t) atomicAdd(&h[t][d], 1u);
            }
          if (pass == 1 && any) {
            const unsigned slot = atomicAdd(&s_ncl, 1u);
            if (slot < RO_CL) s_cl[slot] = k;
          }
        }
      }
      __syncthreads();
      RO_TS(4 + 3 * pass);
      unsigned(*gh)[2048] = sc.hist[pass];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (src[t] != t) continue;
        for (int i = tid; i < 2048; i += RO_TPB) {
          const unsigned v = h[t][i];
          if (v) atomicAdd(&gh[t][i], v);
        }
      }
      RO_TS(5 + 3 * pass);
      ro_barrier(sel, gen0, ++nbar, s_bc, &s_last, [&]() {
        // the last CTA finds, for each target, the digit holding its remaining
        // rank; thread tid owns bins 4 tid .. 4 tid + 3 of each distinct total
        uint4 b[4];
        unsigned sum[4], inc[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          b[t] = src[t] == t ? __ldcg(reinterpret_cast<const uint4 *>(&gh[t][0]) + tid) : make_uint4(0u, 0u, 0u, 0u);
          sum[t] = b[t].x + b[t].y + b[t].z + b[t].w;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          inc[t] = sum[t];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_up_sync(0xffffffffu, inc[t], o);
            if (lane >= o) inc[t] += v;
          }
        }
        if (lane == 31) s_wt[wid] = make_uint4(inc[0], inc[1], inc[2], inc[3]);
        __syncthreads();
        unsigned wofs[4] = {0u, 0u, 0u, 0u};
        for (int w = 0; w < wid; ++w) {
          const uint4 v = s_wt[w];
          wofs[0] += v.x;
          wofs[1] += v.y;
          wofs[2] += v.z;
          wofs[3] += v.w;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          // a duplicate target searches its source's totals (same prefix)
          uint4 bu = b[0];
          unsigned su = sum[0], ex = wofs[0] + inc[0] - sum[0];
#pragma unroll
          for (int u = 1; u < 4; ++u)
            if (src[t] == u) {
              bu = b[u];
              su = sum[u];
              ex = wofs[u] + inc[u] - sum[u];
            }
          if (rank[t] >= ex && rank[t] < ex + su) {
            unsigned q = 0;
            if (rank[t] >= ex + bu.x) {
              ex += bu.x;
              q = 1;
              if (rank[t] >= ex + bu.y) {
                ex += bu.y;
                q = 2;
                if (rank[t] >= ex + bu.z) {
                  ex += bu.z;
                  q = 3;
                }
              }
            }
            const unsigned pf = pref[t] | ((4u * tid + q) << shift);
            sel->bc[t] = pf;
            sel->bc[4 + t] = rank[t] - ex;
          }
        }
      });
      if (tid < 4) {
        s_pref[tid] = s_bc[tid];
        s_rank[tid] = s_bc[4 + tid];
      }
      __syncthreads();
      RO_TS(6 + 3 * pass);
    }
    // numpy _lerp of the two neighbours of each virtual index
    const double a0 = (double)order_unkey(s_pref[0]), b0 = (double)order_unkey(s_pref[1]);
    const double a1 = (double)order_unkey(s_pref[2]), b1 = (double)order_unkey(s_pref[3]);
    const double d0 = __dsub_rn(b0, a0), d1 = __dsub_rn(b1, a1);
    lo = g_lo >= 0.5 ? __dsub_rn(b0, __dmul_rn(d0, __dsub_rn(1.0, g_lo))) : __dadd_rn(a0, __dmul_rn(d0, g_lo));
    hi = g_hi >= 0.5 ? __dsub_rn(b1, __dmul_rn(d1, __dsub_rn(1.0, g_hi))) : __dadd_rn(a1, __dmul_rn(d1, g_hi));
  } else {
    lo = -fixed_bound;
    hi = fixed_bound;
  }
  const bool deg = !(hi > lo);
  if (blockIdx.x == 0 && tid == 0) {
    sel->lo = lo;
    sel->hi = hi;
    sel->degenerate = deg;
    if (robust) sel->parity = par ^ 1u;   // every CTA read it before the first barrier
  }
  const double scale = deg ? 0.0 : __ddiv_rn(255.0, __dsub_rn(hi, lo));
  const bool keys_here = on_chip && robust;
  uint8_t *o = out + beg;
  if ((reinterpret_cast<unsigned long long>(o) & 3ull) == 0 && (keys_here || vec)) {
    for (int i = tid; i < (cnt >> 2); i += RO_TPB) {
      float v[4];
      if (keys_here) {
        const uint4 k = reinterpret_cast<const uint4 *>(ro_keys)[i];
        v[0] = order_unkey(k.x);
        v[1] = order_unkey(k.y);
        v[2] = order_unkey(k.z);
        v[3] = order_unkey(k.w);
      } else {
        const float4 f = __ldcs(reinterpret_cast<const float4 *>(l + beg) + i);
        v[0] = f.x;
        v[1] = f.y;
        v[2] = f.z;
        v[3] = f.w;
      }
      const unsigned w = ro_map(v[0], lo, scale, deg) | (ro_map(v[1], lo, scale, deg) << 8) |
                         (ro_map(v[2], lo, scale, deg) << 16) | (ro_map(v[3], lo, scale, deg) << 24);
      reinterpret_cast<unsigned *>(o)[i] = w;
    }
    for (int i = (cnt & ~3) + tid; i < cnt; i += RO_TPB)
      o[i] = (uint8_t)ro_map(keys_here ? order_unkey(ro_keys[i]) : l[beg + i], lo, scale, deg);
  } else {
    for (int i = tid; i < cnt; i += RO_TPB)
      o[i] = (uint8_t)ro_map(keys_here ? order_unkey(ro_keys[i]) : l[beg + i], lo, scale, deg);
  }
  RO_TS(15);
}

// A snapshot of the brightness for an asynchronous read-out (the read-out then
// runs beside the next batch's blur stage, which rewrites l)
__global__ void __launch_bounds__(TPB) k_snap(const float *__restrict__ src, float *__restrict__ dst, long long n) {
  pdl_wait();
  const long long stride = (long long)gridDim.x * TPB;
  const long long n4 = n >> 2;
  for (long long i = (long long)blockIdx.x * TPB + threadIdx.x; i < n4; i += stride)
    reinterpret_cast<float4 *>(dst)[i] = __ldcg(reinterpret_cast<const float4 *>(src) + i);
  for (long long i = (n4 << 2) + (long long)blockIdx.x * TPB + threadIdx.x; i < n; i += stride) dst[i] = src[i];
}

// ------------------------------------------------------------ EVF1 decode ---

// EVF1 records (event_io.py:60-76): dt u32 LE | xp u16 (bit 15 polarity,
// bits 0..14 x) | y u16.  Two records per thread through one 16-byte load;
// columns out, per-block dt sums for the timestamp scan, first out-of-bounds
// record index (the container is invalid then: DataError, event_io.py:66-72).

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

__global__ void k_init_state(DevState *s, long long q0, BatchState *bs, int nbs) {
  pdl_wait();
  for (int i = 0; i < nbs; ++i) {   // every batch's anchors may start from the initial state
    bs[i].p_s = 0;
    bs[i].p_q = q0;
    bs[i].p_np = 0;
    bs[i].p_nt = 0;
    bs[i].p_geo = 1;
  }
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
__global__ void k_init_pt(PixRec *p, long long *plast, long long n) {
  pdl_wait();
  for (long long i = (long long)blockIdx.x * TPB + threadIdx.x; i < n; i += (long long)gridDim.x * TPB) {
    PixRec r;
    r.st = 0;
    r.end = 0;
    r.carried = FIBAR_NONE;
    r.pad0 = 0;
    p[i] = r;
    plast[i] = -1;
  }
}


}  // namespace fibar
