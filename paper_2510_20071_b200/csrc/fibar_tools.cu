// fibar_tools.cu -- the calibration feeder and the single-pixel trace kernels
// around the hot path:
//
//   fibar_count_events     calib.count_events (calib.py:26-45): per-pixel ON /
//                          OFF event counts, the input of the threshold map whose
//                          gain grid the engine multiplies in (_kernels.py:71-72).
//   fibar_pixel_trace      temporal.stream_pixel -> _kernels.temporal_trace
//                          (_kernels.py:219-233): a pixel's two-stage trajectory.
//   fibar_pixel_trace_iir  temporal.stream_pixel_iir -> _kernels.iir_trace
//                          (_kernels.py:236-249): the combined second-order form.
//
// Counting is HBM-bound integer work: 5 B/event in, a 16 B/pixel table that
// stays in L2 (640x480: 4.9 MB), warp-aggregated atomics so hot pixels do not
// serialise.  A trace is a serial recurrence whose float rounding must match
// the reference's sequential loop bit for bit, so it runs one thread per trace
// (many traces in parallel when the caller passes several).
#include <algorithm>
#include <cstdint>

#include "fibar_common.cuh"
#include "fibar_internal.h"
#include "../../include/fibar_b200.h"

using namespace fibar;

namespace {

constexpr int TPB = 256;

// flat = y*W + x exactly as calib.py:39 forms it (x alone is not range
// checked there: x >= W with flat < n_pix counts into the next row).
__global__ void __launch_bounds__(TPB) k_count_events(const uint16_t *__restrict__ x, const uint16_t *__restrict__ y,
                                                      const int8_t *__restrict__ p, long long n, unsigned W,
                                                      unsigned long long n_pix, unsigned long long *on,
                                                      unsigned long long *off, unsigned long long *bad) {
  const unsigned lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * TPB;
  // whole warps iterate together so the match below always sees a full warp
  const long long n_round = (n + 31) & ~31LL;
  for (long long i = (long long)blockIdx.x * TPB + threadIdx.x; i < n_round; i += stride) {
    bool ok = false;
    unsigned long long key = ~0ull;
    if (i < n) {
      const unsigned long long flat = (unsigned long long)y[i] * W + x[i];
      if (flat >= n_pix) {
        atomicMin(bad, (unsigned long long)i);
      } else {
        ok = true;
        key = flat * 2 + (p[i] > 0 ? 1 : 0);
      }
    }
    // warp aggregation: one atomic per distinct (pixel, polarity) in the warp
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (ok && lane == (unsigned)(__ffs(peers) - 1)) {
      unsigned long long *dst = (key & 1) ? on : off;
      atomicAdd(dst + (key >> 1), (unsigned long long)__popc(peers));
    }
  }
}

template <class T>
struct Ar;
template <>
struct Ar<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
};
template <>
struct Ar<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
};

// _kernels.py:219-233, one thread per trace; separately rounded operations in
// the reference's order: pb = a*pb + (1-a)*p; d = p - pb; l = b*l + h*d.
template <class T>
__global__ void k_trace(const int8_t *__restrict__ ps, long long n, int ntr, T a, T oma, T b, T h, T *state, T *opb,
                        T *od, T *ol) {
  const int tr = blockIdx.x * blockDim.x + threadIdx.x;
  if (tr >= ntr) return;
  const long long base = (long long)tr * n;
  T pb = state[2 * tr], lv = state[2 * tr + 1];
  for (long long j = 0; j < n; ++j) {
    const T pv = (T)ps[base + j];
    pb = Ar<T>::add(Ar<T>::mul(a, pb), Ar<T>::mul(oma, pv));
    const T d = Ar<T>::sub(pv, pb);
    lv = Ar<T>::add(Ar<T>::mul(b, lv), Ar<T>::mul(h, d));
    opb[base + j] = pb;
    od[base + j] = d;
    ol[base + j] = lv;
  }
  state[2 * tr] = pb;
  state[2 * tr + 1] = lv;
}

// _kernels.py:236-249: l = ((a+b)*l1 - (a*b)*l2) + h*(p - p_prev)
template <class T>
__global__ void k_trace_iir(const int8_t *__restrict__ ps, long long n, int ntr, T apb, T atb, T h, T *state,
                            T *ol) {
  const int tr = blockIdx.x * blockDim.x + threadIdx.x;
  if (tr >= ntr) return;
  const long long base = (long long)tr * n;
  T l1 = state[3 * tr], l2 = state[3 * tr + 1], pp = state[3 * tr + 2];
  for (long long j = 0; j < n; ++j) {
    const T pv = (T)ps[base + j];
    const T lv = Ar<T>::add(Ar<T>::sub(Ar<T>::mul(apb, l1), Ar<T>::mul(atb, l2)), Ar<T>::mul(h, Ar<T>::sub(pv, pp)));
    ol[base + j] = lv;
    l2 = l1;
    l1 = lv;
    pp = pv;
  }
  state[3 * tr] = l1;
  state[3 * tr + 1] = l2;
  state[3 * tr + 2] = pp;
}

}  // namespace

extern "C" {

int fibar_count_events(const uint16_t *x, const uint16_t *y, const int8_t *p, int64_t n, int32_t width, int64_t n_pix,
                       int64_t *n_on, int64_t *n_off, int64_t *first_bad, void *stream) {
  if (n < 0 || width < 1 || n_pix < 1 || !n_on || !n_off || !first_bad) return fail(FIBAR_E_CONFIG, "bad arguments");
  *first_bad = -1;
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  unsigned long long *bad = nullptr;
  CK(cudaMallocAsync((void **)&bad, sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), s));
  const long long want = (n + TPB - 1) / TPB;
  const int grid = (int)std::min<long long>(want, (long long)nsm * 8);
  k_count_events<<<grid, TPB, 0, s>>>(x, y, p, n, (unsigned)width, (unsigned long long)n_pix,
                                      reinterpret_cast<unsigned long long *>(n_on),
                                      reinterpret_cast<unsigned long long *>(n_off), bad);
  CK(cudaGetLastError());
  unsigned long long hb = 0;
  CK(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(bad, s);
  CK(cudaStreamSynchronize(s));
  *first_bad = hb == ~0ull ? -1 : (int64_t)hb;
  return 0;
}

int fibar_pixel_trace(const int8_t *p, int64_t n, int32_t ntraces, int32_t dtype, const double coef[4], void *state,
                      void *p_bar, void *delta, void *l, void *stream) {
  if (n < 0 || ntraces < 0 || !coef || (dtype != 0 && dtype != 1)) return fail(FIBAR_E_CONFIG, "bad arguments");
  if (n == 0 || ntraces == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int blocks = (ntraces + 127) / 128;
  if (dtype == 0)
    k_trace<float><<<blocks, 128, 0, s>>>(p, n, ntraces, (float)coef[0], (float)coef[1], (float)coef[2],
                                          (float)coef[3], (float *)state, (float *)p_bar, (float *)delta, (float *)l);
  else
    k_trace<double><<<blocks, 128, 0, s>>>(p, n, ntraces, coef[0], coef[1], coef[2], coef[3], (double *)state,
                                           (double *)p_bar, (double *)delta, (double *)l);
  CK(cudaGetLastError());
  return 0;
}

int fibar_pixel_trace_iir(const int8_t *p, int64_t n, int32_t ntraces, int32_t dtype, const double coef[3],
                          void *state, void *l, void *stream) {
  if (n < 0 || ntraces < 0 || !coef || (dtype != 0 && dtype != 1)) return fail(FIBAR_E_CONFIG, "bad arguments");
  if (n == 0 || ntraces == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int blocks = (ntraces + 127) / 128;
  if (dtype == 0)
    k_trace_iir<float><<<blocks, 128, 0, s>>>(p, n, ntraces, (float)coef[0], (float)coef[1], (float)coef[2],
                                              (float *)state, (float *)l);
  else
    k_trace_iir<double><<<blocks, 128, 0, s>>>(p, n, ntraces, coef[0], coef[1], coef[2], (double *)state,
                                               (double *)l);
  CK(cudaGetLastError());
  return 0;
}

}  // extern "C"
