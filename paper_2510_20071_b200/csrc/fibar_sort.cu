// fibar_sort.cu -- stable LSD radix sort of (tile-major pixel key, event index)
// pairs for one device batch.  Digits of up to 10 bits (20 key bits: two
// passes of 10 instead of three of 8), 2048-item tiles per CTA.
//
// Role on the path: groups a batch's events by pixel (and, because the key is
// tile-major, by 2x2 tile) while keeping each pixel's events in stream order --
// the order the reference's per-event loop visits them (_kernels.py:119-130).
//
// The batch size lives in device memory (after OOB compaction), so every
// kernel is launched for the host-side upper bound and reads the real count.
#include "fibar_common.cuh"
#include "fibar_internal.h"

namespace fibar {

constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 8;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 2048
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_MAX_BITS = 10;               // widest digit (per-warp counters: 8 x 1024 x 4 B of shared memory)
constexpr int RS_MAX_BINS = 1 << RS_MAX_BITS;

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const unsigned *__restrict__ keys,
                                                         const long long *__restrict__ n_dev, int shift, int dbits,
                                                         unsigned *__restrict__ hist, int nblocks) {
  pdl_wait();
  __shared__ unsigned h[RS_MAX_BINS];
  const long long n = *n_dev;
  const int bins = 1 << dbits;
  const unsigned dmask = (unsigned)bins - 1u;
  for (int i = threadIdx.x; i < bins; i += RS_THREADS) h[i] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * RS_TILE;
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    long long i = base + r * RS_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & dmask], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < bins; d += RS_THREADS) hist[(long long)d * nblocks + blockIdx.x] = h[d];
}

// exclusive scan of `len` counters in place with one CTA of 1024 threads,
// 16 counters per thread per round (uint4 loads when aligned)
__global__ void __launch_bounds__(1024) k_scan_inplace(unsigned *__restrict__ a, int len) {
  pdl_wait();
  constexpr int PER = 16;
  __shared__ unsigned warp_tot[32];
  __shared__ unsigned carry_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (len > 1024 * PER && (reinterpret_cast<uintptr_t>(a) & 15) == 0) {
    // more than one round's worth (the 10-bit radix histograms of a small
    // batch: 64k counters): every warp takes one contiguous span, a multiple
    // of 128 counters, read with coalesced 16-byte loads.  Pass 1 sums the
    // spans, the block scans the 32 sums once, pass 2 rewrites each span as
    // prefixes, 128 counters per step with the next step's load in flight --
    // two barriers in all instead of two per 16k counters.
    const int span = (((len + 31) / 32) + 127) & ~127;
    const int w0 = wid * span, w1 = min(len, w0 + span);
    const int nfull = max(0, w1 - w0) >> 7;   // steps of 128 counters with every lane in range
    unsigned tsum = 0;
    {
      int it = 0;
      for (; it + 4 <= nfull; it += 4) {
        uint4 q[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) q[r] = *reinterpret_cast<const uint4 *>(a + w0 + (it + r) * 128 + lane * 4);
#pragma unroll
        for (int r = 0; r < 4; ++r) tsum += q[r].x + q[r].y + q[r].z + q[r].w;
      }
      for (; it < nfull; ++it) {
        const uint4 q = *reinterpret_cast<const uint4 *>(a + w0 + it * 128 + lane * 4);
        tsum += q.x + q.y + q.z + q.w;
      }
      for (int i = w0 + nfull * 128 + lane; i < w1; i += 32) tsum += a[i];   // the array's ragged end
    }
    tsum = __reduce_add_sync(0xffffffffu, tsum);
    if (lane == 0) warp_tot[wid] = tsum;
    __syncthreads();
    if (wid == 0) {
      const unsigned w = warp_tot[lane];
      unsigned wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      warp_tot[lane] = wi - w;
    }
    __syncthreads();
    unsigned run = warp_tot[wid];   // exclusive prefix of the span
    uint4 nxt = nfull > 0 ? *reinterpret_cast<const uint4 *>(a + w0 + lane * 4) : make_uint4(0u, 0u, 0u, 0u);
    for (int it = 0; it < nfull; ++it) {
      const uint4 q = nxt;
      if (it + 1 < nfull) nxt = *reinterpret_cast<const uint4 *>(a + w0 + (it + 1) * 128 + lane * 4);
      const unsigned ts = q.x + q.y + q.z + q.w;
      unsigned incl = ts;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const unsigned r0 = run + incl - ts, r1 = r0 + q.x, r2 = r1 + q.y, r3 = r2 + q.z;
      *reinterpret_cast<uint4 *>(a + w0 + it * 128 + lane * 4) = make_uint4(r0, r1, r2, r3);
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    // the ragged end (fewer than 128 counters, the last warp in range only): lane 0 finishes it
    if (lane == 0)
      for (int i = w0 + nfull * 128; i < w1; ++i) {
        const unsigned t = a[i];
        a[i] = run;
        run += t;
      }
    return;
  }
  unsigned carry = 0;
  for (int base = 0; base < len; base += 1024 * PER) {
    unsigned v[PER];
    const int i0 = base + threadIdx.x * PER;
    if (i0 + PER <= len && ((reinterpret_cast<uintptr_t>(a + i0) & 15) == 0)) {
#pragma unroll
      for (int r = 0; r < PER / 4; ++r) {
        const uint4 q = reinterpret_cast<const uint4 *>(a + i0)[r];
        v[4 * r] = q.x;
        v[4 * r + 1] = q.y;
        v[4 * r + 2] = q.z;
        v[4 * r + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int r = 0; r < PER; ++r) v[r] = i0 + r < len ? a[i0 + r] : 0u;
    }
    unsigned tsum = 0;
#pragma unroll
    for (int r = 0; r < PER; ++r) tsum += v[r];
    unsigned incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const unsigned w = warp_tot[lane];
      unsigned wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      warp_tot[lane] = wi - w;
      if (lane == 31) carry_s = wi;
    }
    __syncthreads();
    unsigned run = carry + warp_tot[wid] + incl - tsum;
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const unsigned t = v[r];
      v[r] = run;
      run += t;
    }
    if (i0 + PER <= len && ((reinterpret_cast<uintptr_t>(a + i0) & 15) == 0)) {
#pragma unroll
      for (int r = 0; r < PER / 4; ++r)
        reinterpret_cast<uint4 *>(a + i0)[r] = make_uint4(v[4 * r], v[4 * r + 1], v[4 * r + 2], v[4 * r + 3]);
    } else {
#pragma unroll
      for (int r = 0; r < PER; ++r)
        if (i0 + r < len) a[i0 + r] = v[r];
    }
    carry += carry_s;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const unsigned *__restrict__ kin,
                                                            const unsigned *__restrict__ vin,
                                                            unsigned *__restrict__ kout, unsigned *__restrict__ vout,
                                                            const long long *__restrict__ n_dev, int shift, int dbits,
                                                            const unsigned *__restrict__ hist, int nblocks) {
  pdl_wait();
  __shared__ unsigned wcnt_s[RS_WARPS * RS_MAX_BINS];
  const long long n = *n_dev;
  const int bins = 1 << dbits;
  const unsigned dmask = (unsigned)bins - 1u;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned *wcnt_w = wcnt_s + wid * bins;   // this warp's counters
  for (int i = threadIdx.x; i < RS_WARPS * bins; i += RS_THREADS) wcnt_s[i] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * RS_TILE + (long long)wid * (RS_ITEMS * 32);
  unsigned key[RS_ITEMS], val[RS_ITEMS], loc[RS_ITEMS];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    long long i = base + r * 32 + lane;
    bool valid = i < n;
    unsigned vmask = __ballot_sync(0xffffffffu, valid);
    key[r] = valid ? kin[i] : 0u;
    val[r] = valid ? (vin ? vin[i] : (unsigned)i) : 0u;
    unsigned d = (key[r] >> shift) & dmask;
    if (valid) {
      unsigned peers = __match_any_sync(vmask, d);
      unsigned before = wcnt_w[d];
      loc[r] = before + __popc(peers & lt);
      __syncwarp(vmask);
      if ((peers & lt) == 0) wcnt_w[d] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // exclusive prefix over warps, per digit
  for (int d = threadIdx.x; d < bins; d += RS_THREADS) {
    unsigned run = hist[(long long)d * nblocks + blockIdx.x];
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
      unsigned t = wcnt_s[w * bins + d];
      wcnt_s[w * bins + d] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    long long i = base + r * 32 + lane;
    if (i < n) {
      unsigned d = (key[r] >> shift) & dmask;
      unsigned pos = wcnt_w[d] + loc[r];
      kout[pos] = key[r];
      vout[pos] = val[r];
    }
  }
}

// A tiny batch (up to one tile of 2048 pairs) sorted by one CTA in shared
// memory: the same stable LSD passes (8-bit digits, match_any ranks in a warp,
// per-warp counters, warps in item order) without leaving the chip -- one
// launch instead of three per pass.  Keys in, (keys, original index) out.
__global__ void __launch_bounds__(RS_THREADS) k_sort_tiny(const unsigned *__restrict__ kin, unsigned *__restrict__ kout,
                                                          unsigned *__restrict__ vout,
                                                          const long long *__restrict__ n_dev, int bits) {
  pdl_wait();
  __shared__ unsigned sk[2][RS_TILE], sv[2][RS_TILE];
  __shared__ unsigned wcnt[RS_WARPS][256];
  __shared__ unsigned wtot[RS_WARPS];
  const int n = (int)min((long long)RS_TILE, *n_dev);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < n; i += RS_THREADS) {
    sk[0][i] = kin[i];
    sv[0][i] = (unsigned)i;
  }
  int cur = 0;
  const unsigned lt = (1u << lane) - 1u;
  const int base = wid * (RS_ITEMS * 32);
  for (int shift = 0; shift < bits; shift += 8) {
    for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    unsigned key[RS_ITEMS], val[RS_ITEMS], loc[RS_ITEMS];
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
      const int i = base + r * 32 + lane;
      const bool valid = i < n;
      const unsigned vmask = __ballot_sync(0xffffffffu, valid);
      key[r] = valid ? sk[cur][i] : 0u;
      val[r] = valid ? sv[cur][i] : 0u;
      const unsigned d = (key[r] >> shift) & 255u;
      if (valid) {
        const unsigned peers = __match_any_sync(vmask, d);
        const unsigned before = wcnt[wid][d];
        loc[r] = before + __popc(peers & lt);
        __syncwarp(vmask);
        if ((peers & lt) == 0) wcnt[wid][d] = before + __popc(peers);
      }
      __syncwarp();
    }
    __syncthreads();
    {
      // digit d = threadIdx.x: exclusive prefix over (digit, warp)
      const int d = threadIdx.x;
      unsigned tot = 0;
#pragma unroll
      for (int w = 0; w < RS_WARPS; ++w) tot += wcnt[w][d];
      unsigned incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wtot[wid] = incl;
      __syncthreads();
      unsigned run = incl - tot;
      for (int w = 0; w < wid; ++w) run += wtot[w];
#pragma unroll
      for (int w = 0; w < RS_WARPS; ++w) {
        const unsigned t = wcnt[w][d];
        wcnt[w][d] = run;
        run += t;
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ITEMS; ++r) {
      const int i = base + r * 32 + lane;
      if (i < n) {
        const unsigned d = (key[r] >> shift) & 255u;
        const unsigned pos = wcnt[wid][d] + loc[r];
        sk[cur ^ 1][pos] = key[r];
        sv[cur ^ 1][pos] = val[r];
      }
    }
    cur ^= 1;
    __syncthreads();
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += RS_THREADS) {
    kout[i] = sk[cur][i];
    vout[i] = sv[cur][i];
  }
}

// Sort (keys, index) for n_dev (<= n_max) items; `bits` significant key bits.
// Pass 0 reads k_a with implicit identity payload; passes alternate between
// the (a) and (b) buffers.  Returns 0 if the result is in (k_a, v_a), 1 if in
// (k_b, v_b).
int radix_sort_pairs(Launcher &L, unsigned *k_a, unsigned *v_a, unsigned *k_b, unsigned *v_b, unsigned *hist,
                     const long long *n_dev, long long n_max, int bits) {
  const int nblocks = (int)((n_max + RS_TILE - 1) / RS_TILE);
  if (n_max > 0 && n_max <= RS_TILE) {   // one tile: sorted on chip by one CTA, result in (k_b, v_b)
    fibar_launch(L, "sort_tiny", k_sort_tiny, 1, RS_THREADS, 0, L.stream, (const unsigned *)k_a, k_b, v_b, n_dev, bits);
    return 1;
  }
  // the fewest passes with digits of at most RS_MAX_BITS bits, the digits as narrow as that allows
  const int passes = bits <= 0 ? 1 : (bits + RS_MAX_BITS - 1) / RS_MAX_BITS;
  const int dbits = bits <= 0 ? 1 : (bits + passes - 1) / passes;
  const long long bins = 1LL << dbits;
  if (nblocks == 0) return 0;
  for (int ps = 0; ps < passes; ++ps) {
    const int shift = ps * dbits;
    const bool a_to_b = (ps % 2) == 0;
    const unsigned *ki = a_to_b ? k_a : k_b;
    const unsigned *vi = ps == 0 ? nullptr : (a_to_b ? v_a : v_b);
    unsigned *ko = a_to_b ? k_b : k_a;
    unsigned *vo = a_to_b ? v_b : v_a;
    fibar_launch(L, "rs_hist", k_rs_hist, nblocks, RS_THREADS, 0, L.stream, ki, n_dev, shift, dbits, hist, nblocks);
    if (bins * nblocks <= 1024 * 16 * 4)   // small sorts: one single-block scan kernel instead of three
      scan_exclusive_u32(L, hist, (int)(bins * nblocks));
    else
      scan_exclusive_large(L, hist, hist, nullptr, bins * nblocks, bins * nblocks, hist + bins * nblocks);
    fibar_launch(L, "rs_scatter", k_rs_scatter, nblocks, RS_THREADS, 0, L.stream, ki, vi, ko, vo, n_dev, shift, dbits, hist,
                 nblocks);
  }
  return (passes % 2) == 1 ? 1 : 0;
}

// --- multi-block exclusive scan (reduce / scan partials / scan + offset) ---
constexpr int SC_THREADS = 256, SC_PER = 16, SC_TILE = SC_THREADS * SC_PER;  // 4096 per block

__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned *wsum, unsigned &total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const unsigned w = lane < SC_THREADS / 32 ? wsum[lane] : 0u;
    unsigned wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < SC_THREADS / 32) wsum[lane] = wi - w;
    if (lane == SC_THREADS / 32 - 1) wsum[SC_THREADS / 32] = wi;
  }
  __syncthreads();
  total = wsum[SC_THREADS / 32];
  return wsum[wid] + inc - v;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_reduce(const unsigned *__restrict__ in, const long long *n_dev,
                                                            long long n_fixed, unsigned *__restrict__ part) {
  pdl_wait();
  __shared__ unsigned wsum[SC_THREADS / 32 + 1];
  const long long n = n_dev ? *n_dev : n_fixed;
  const long long i0 = (long long)blockIdx.x * SC_TILE + threadIdx.x * SC_PER;
  unsigned v = 0;
#pragma unroll
  for (int r = 0; r < SC_PER; ++r)
    if (i0 + r < n) v += in[i0 + r];
  unsigned tot;
  block_excl_scan(v, wsum, tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_apply(const unsigned *__restrict__ in, unsigned *__restrict__ out,
                                                           const long long *n_dev, long long n_fixed,
                                                           const unsigned *__restrict__ part) {
  pdl_wait();
  __shared__ unsigned wsum[SC_THREADS / 32 + 1];
  const long long n = n_dev ? *n_dev : n_fixed;
  const long long i0 = (long long)blockIdx.x * SC_TILE + threadIdx.x * SC_PER;
  unsigned v[SC_PER];
  unsigned t = 0;
#pragma unroll
  for (int r = 0; r < SC_PER; ++r) {
    v[r] = i0 + r < n ? in[i0 + r] : 0u;
    t += v[r];
  }
  unsigned tot;
  unsigned run = part[blockIdx.x] + block_excl_scan(t, wsum, tot);
#pragma unroll
  for (int r = 0; r < SC_PER; ++r) {
    if (i0 + r < n) out[i0 + r] = run;
    run += v[r];
  }
}

// exclusive scan of n (device count, or n_fixed when n_dev is null) counters,
// n <= n_max; part needs n_max / 4096 + 2 entries
void scan_exclusive_large(Launcher &L, const unsigned *in, unsigned *out, const long long *n_dev, long long n_fixed,
                          long long n_max, unsigned *part) {
  const int nb = (int)((n_max + SC_TILE - 1) / SC_TILE);
  if (nb == 0) return;
  fibar_launch(L, "scan_reduce", k_scan_reduce, nb, SC_THREADS, 0, L.stream, in, n_dev, n_fixed, part);
  fibar_launch(L, "scan", k_scan_inplace, 1, 1024, 0, L.stream, part, nb);
  fibar_launch(L, "scan_apply", k_scan_apply, nb, SC_THREADS, 0, L.stream, in, out, n_dev, n_fixed, part);
}

void scan_exclusive_u32(Launcher &L, unsigned *a, int len) {
  fibar_launch(L, "scan", k_scan_inplace, 1, 1024, 0, L.stream, a, len);
}

}  // namespace fibar
