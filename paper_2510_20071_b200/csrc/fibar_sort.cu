// fibar_sort.cu -- stable LSD radix sort of (tile-major pixel key, event index)
// pairs for one device batch.  8-bit digits, 2048-item tiles per CTA.
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

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const unsigned *__restrict__ keys,
                                                         const long long *__restrict__ n_dev, int shift,
                                                         unsigned *__restrict__ hist, int nblocks) {
  pdl_wait();
  __shared__ unsigned h[256];
  const long long n = *n_dev;
  for (int i = threadIdx.x; i < 256; i += RS_THREADS) h[i] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * RS_TILE;
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    long long i = base + r * RS_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += RS_THREADS) hist[(long long)d * nblocks + blockIdx.x] = h[d];
}

// exclusive scan of `len` counters in place with one CTA of 1024 threads,
// 16 counters per thread per round (uint4 loads when aligned)
__global__ void __launch_bounds__(1024) k_scan_inplace(unsigned *__restrict__ a, int len) {
  pdl_wait();
  constexpr int PER = 16;
  __shared__ unsigned warp_tot[32];
  __shared__ unsigned carry_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
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
                                                            const long long *__restrict__ n_dev, int shift,
                                                            const unsigned *__restrict__ hist, int nblocks) {
  pdl_wait();
  __shared__ unsigned wcnt[RS_WARPS][256];
  const long long n = *n_dev;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&wcnt[0][0])[i] = 0;
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
    unsigned d = (key[r] >> shift) & 255u;
    if (valid) {
      unsigned peers = __match_any_sync(vmask, d);
      unsigned before = wcnt[wid][d];
      loc[r] = before + __popc(peers & lt);
      __syncwarp(vmask);
      if ((peers & lt) == 0) wcnt[wid][d] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // exclusive prefix over warps, per digit
  for (int d = threadIdx.x; d < 256; d += RS_THREADS) {
    unsigned run = hist[(long long)d * nblocks + blockIdx.x];
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
      unsigned t = wcnt[w][d];
      wcnt[w][d] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    long long i = base + r * 32 + lane;
    if (i < n) {
      unsigned d = (key[r] >> shift) & 255u;
      unsigned pos = wcnt[wid][d] + loc[r];
      kout[pos] = key[r];
      vout[pos] = val[r];
    }
  }
}

// Sort (keys, index) for n_dev (<= n_max) items; `bits` significant key bits.
// Pass 0 reads k_a with implicit identity payload; passes alternate between
// the (a) and (b) buffers.  Returns 0 if the result is in (k_a, v_a), 1 if in
// (k_b, v_b).
int radix_sort_pairs(Launcher &L, unsigned *k_a, unsigned *v_a, unsigned *k_b, unsigned *v_b, unsigned *hist,
                     const long long *n_dev, long long n_max, int bits) {
  const int nblocks = (int)((n_max + RS_TILE - 1) / RS_TILE);
  const int passes = bits <= 0 ? 1 : (bits + 7) / 8;
  if (nblocks == 0) return 0;
  for (int ps = 0; ps < passes; ++ps) {
    const int shift = ps * 8;
    const bool a_to_b = (ps % 2) == 0;
    const unsigned *ki = a_to_b ? k_a : k_b;
    const unsigned *vi = ps == 0 ? nullptr : (a_to_b ? v_a : v_b);
    unsigned *ko = a_to_b ? k_b : k_a;
    unsigned *vo = a_to_b ? v_b : v_a;
    fibar_launch(L, "rs_hist", k_rs_hist, nblocks, RS_THREADS, 0, L.stream, ki, n_dev, shift, hist, nblocks);
    if (256LL * nblocks <= 1024 * 16)   // small sorts: one single-pass scan kernel instead of three
      scan_exclusive_u32(L, hist, 256 * nblocks);
    else
      scan_exclusive_large(L, hist, hist, nullptr, 256LL * nblocks, 256LL * nblocks, hist + 256LL * nblocks);
    fibar_launch(L, "rs_scatter", k_rs_scatter, nblocks, RS_THREADS, 0, L.stream, ki, vi, ko, vo, n_dev, shift, hist, nblocks);
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
