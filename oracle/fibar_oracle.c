/*
 * fibar_oracle.c -- CPU restatement of the FIBAR reconstruction hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path; it is never linked into, called by, or shipped with the product
 * library (paper_2510_20071_b200/_lib/libfibar_b200.so).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.
 *
 * Every routine restates the reference algorithm in plain C, strict IEEE
 * float32 with no contraction (build with -ffp-contract=off), so that it
 * agrees bit for bit with the reference's numba kernels.  Parity of this
 * restatement is pinned against golden vectors produced by running the
 * reference itself (tests/golden/make_golden.py, tests/test_oracle_golden.py).
 *
 * Reference map (paths relative to /root/reference/pkg/src/fibar):
 *   oracle_temporal_chunk  <- _kernels.py:62-73   (_temporal_chunk)
 *   oracle_full_chunk      <- _kernels.py:76-216  (_full_chunk), QS_* slots 48-59
 *   oracle_blur_at         <- _kernels.py:252-268 (_blur_at)
 *   oracle_render          <- pipeline.py:247-269 (render) + numpy 2.3.5
 *                             percentile 'linear' (virtual index (n-1)q, _lerp)
 *   oracle_decode_evf1     <- event_io.py:60-76 (_decode_block)
 *   oracle_trace_f32/_f64  <- _kernels.py:219-233 (_temporal_trace)
 *   oracle_trace_iir_f32/_f64 <- _kernels.py:236-249 (_iir_trace)
 *   oracle_count_events    <- calib.py:26-45 (count_events, flat = y*W + x)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum {
  Q_HEAD = 0, Q_LEN, Q_TARGET, Q_NPIX, Q_NTILES, Q_BLUR, Q_STALE, Q_QTMIN,
  Q_QTMAX, Q_EVCTR, Q_SLOTS
};

/* Per-event two-stage filter, temporal path only (_kernels.py:62-73). */
void oracle_temporal_chunk(const uint16_t *xs, const uint16_t *ys,
                           const int8_t *ps, int64_t n, int64_t width,
                           float *p_bar, float *l, float alpha,
                           float one_m_alpha, float beta, float half_1p_beta,
                           const float *gain, int use_gain) {
  for (int64_t e = 0; e < n; ++e) {
    int64_t pix = (int64_t)ys[e] * width + (int64_t)xs[e];
    float pol = (float)ps[e];
    float a = alpha * p_bar[pix];
    float b = one_m_alpha * pol;
    float avg = a + b;
    p_bar[pix] = avg;
    float inc = pol - avg;
    if (use_gain) inc = inc * gain[pix];
    float lb = beta * l[pix];
    float hb = half_1p_beta * inc;
    l[pix] = lb + hb;
  }
}

/* Renormalised 3x3 binomial blur value at (x, y) (_kernels.py:252-268).
 * Taps in dy-outer / dx-inner order, out-of-bounds taps skipped. */
float oracle_blur_at(const float *l, int64_t width, int64_t height, int64_t x,
                     int64_t y) {
  float num = 0.0f, den = 0.0f;
  for (int dy = -1; dy <= 1; ++dy) {
    int64_t yy = y + dy;
    if (yy < 0 || yy >= height) continue;
    int wy = dy == 0 ? 2 : 1;
    for (int dx = -1; dx <= 1; ++dx) {
      int64_t xx = x + dx;
      if (xx < 0 || xx >= width) continue;
      float w = (float)(wy * (dx == 0 ? 2 : 1));
      float prod = w * l[yy * width + xx];
      num = num + prod;
      den = den + w;
    }
  }
  return num / den;
}

/* Fused temporal + active-window tracking + stale blur (_kernels.py:76-216).
 *
 * Optional instrumentation (any pointer may be NULL):
 *   stale_k / stale_j : for every staleness episode, the in-bounds index of
 *                       the popped event k and of the event j whose trim
 *                       popped it, both counted from ev_base (the number of
 *                       in-bounds events the engine had consumed before this
 *                       call).  Capacity stale_cap; *n_stale receives the
 *                       number of episodes (which may exceed the capacity;
 *                       entries beyond it are not written).
 * The ring slot of an event is its in-bounds index mod qcap. */
void oracle_full_chunk(const uint16_t *xs, const uint16_t *ys,
                       const int8_t *ps, int64_t n, int64_t width,
                       int64_t height, int64_t tiles_x, int64_t tile_side,
                       int64_t area, float *p_bar, float *l,
                       uint16_t *active_count, uint8_t *tile_count,
                       uint16_t *qx, uint16_t *qy, int64_t qcap, int64_t *qs,
                       float alpha, float one_m_alpha, float beta,
                       float half_1p_beta, const float *gain, int use_gain,
                       int64_t fill_num, int64_t fill_den, int64_t q_min,
                       int64_t q_max, int blur_on, int64_t regulate_every,
                       int64_t ev_base, int64_t *stale_k, int64_t *stale_j,
                       int64_t stale_cap, int64_t *n_stale) {
  int64_t head = qs[Q_HEAD], qlen = qs[Q_LEN], target = qs[Q_TARGET];
  int64_t npix = qs[Q_NPIX], ntiles = qs[Q_NTILES];
  int64_t blurs = qs[Q_BLUR], stales = qs[Q_STALE];
  int64_t tmin = qs[Q_QTMIN], tmax = qs[Q_QTMAX], evctr = qs[Q_EVCTR];
  int64_t recorded = 0;

  for (int64_t e = 0; e < n; ++e) {
    const int64_t x = xs[e], y = ys[e];
    const int64_t pix = y * width + x;

    /* temporal update, identical arithmetic to the filter-off path */
    float pol = (float)ps[e];
    float a = alpha * p_bar[pix];
    float b = one_m_alpha * pol;
    float avg = a + b;
    p_bar[pix] = avg;
    float inc = pol - avg;
    if (use_gain) inc = inc * gain[pix];
    float lb = beta * l[pix];
    float hb = half_1p_beta * inc;
    l[pix] = lb + hb;

    /* push to the back of the ring */
    int64_t slot = head + qlen;
    if (slot >= qcap) slot -= qcap;
    qx[slot] = (uint16_t)x;
    qy[slot] = (uint16_t)y;
    ++qlen;
    const int64_t cnt = active_count[pix];
    if (cnt == 0) {
      ++npix;
      const int64_t tile = (y / tile_side) * tiles_x + (x / tile_side);
      const int64_t tc = tile_count[tile];
      if (tc == 0) ++ntiles;
      if (tc < 255) tile_count[tile] = (uint8_t)(tc + 1);
    }
    if (cnt < 65535) active_count[pix] = (uint16_t)(cnt + 1);

    /* pop the front down to the current target */
    while (qlen > target) {
      const int64_t px = qx[head], py = qy[head];
      const int64_t popped_slot_index = ev_base + e - qlen + 1;
      ++head;
      if (head >= qcap) head -= qcap;
      --qlen;
      const int64_t ppix = py * width + px;
      int64_t c2 = active_count[ppix];
      if (c2 <= 0) continue;
      --c2;
      active_count[ppix] = (uint16_t)c2;
      if (c2 != 0) continue;
      ++stales;
      --npix;
      const int64_t tile = (py / tile_side) * tiles_x + (px / tile_side);
      const int64_t tc = tile_count[tile];
      if (tc > 0) {
        tile_count[tile] = (uint8_t)(tc - 1);
        if (tc == 1) --ntiles;
      }
      if (stale_k && recorded < stale_cap) {
        stale_k[recorded] = popped_slot_index;
        stale_j[recorded] = ev_base + e;
      }
      ++recorded;
      if (blur_on) {
        l[ppix] = oracle_blur_at(l, width, height, px, py);
        ++blurs;
      }
    }

    /* integer fill-ratio regulation */
    if (++evctr >= regulate_every) {
      evctr = 0;
      if (npix >= 1 && ntiles >= 1) {
        int64_t want = (qlen * fill_num * ntiles * area) / (fill_den * npix);
        if (want < q_min) want = q_min;
        if (want > q_max) want = q_max;
        target = want;
        if (target < tmin) tmin = target;
        if (target > tmax) tmax = target;
      }
    }
  }
  qs[Q_HEAD] = head; qs[Q_LEN] = qlen; qs[Q_TARGET] = target;
  qs[Q_NPIX] = npix; qs[Q_NTILES] = ntiles; qs[Q_BLUR] = blurs;
  qs[Q_STALE] = stales; qs[Q_QTMIN] = tmin; qs[Q_QTMAX] = tmax;
  qs[Q_EVCTR] = evctr;
  if (n_stale) *n_stale = recorded;
}

/* ---- read-out ---------------------------------------------------------- */

static void swap_d(double *a, double *b) { double t = *a; *a = *b; *b = t; }

/* k-th smallest (0-based) by iterative quickselect with median-of-three.
 * Equal values are interchangeable, so any correct selection gives the
 * value numpy's introselect partition places at index k. */
static double select_kth(double *v, int64_t n, int64_t k) {
  int64_t lo = 0, hi = n - 1;
  while (hi > lo) {
    int64_t mid = lo + (hi - lo) / 2;
    if (v[mid] < v[lo]) swap_d(&v[mid], &v[lo]);
    if (v[hi] < v[lo]) swap_d(&v[hi], &v[lo]);
    if (v[hi] < v[mid]) swap_d(&v[hi], &v[mid]);
    double pivot = v[mid];
    int64_t i = lo, j = hi;
    while (i <= j) {
      while (v[i] < pivot) ++i;
      while (v[j] > pivot) --j;
      if (i <= j) { swap_d(&v[i], &v[j]); ++i; --j; }
    }
    if (k <= j) hi = j;
    else if (k >= i) lo = i;
    else return v[k];
  }
  return v[k];
}

/* numpy 'linear' percentile of float64 data: virtual index (n-1)*q,
 * neighbours floor / floor+1 clamped at the top, then numpy's _lerp
 * (a + d*g, or b - d*(1-g) when g >= 0.5). */
static double percentile_linear(double *work, int64_t n, double q) {
  double vidx = (double)(n - 1) * q;
  int64_t prev, next;
  if (vidx >= (double)(n - 1)) {
    prev = next = n - 1;
  } else if (vidx < 0) {
    prev = next = 0;
  } else {
    prev = (int64_t)floor(vidx);
    next = prev + 1;
  }
  double gamma = vidx - (double)prev;
  double a = select_kth(work, n, prev);
  double b = select_kth(work, n, next);
  double d = b - a;
  double r = a + d * gamma;
  if (gamma >= 0.5) r = b - d * (1.0 - gamma);
  return r;
}

/* render (pipeline.py:247-269).  mode 0 = robust (1st..99th percentile),
 * 1 = fixed (+-bound).  Writes n uint8 pixels, bounds[2], *degenerate.
 * Returns 0, or -1 on a bad mode / bound (the caller raises ConfigError). */
int oracle_render(const float *l, int64_t n, int mode, double fixed_bound,
                  uint8_t *out, double *bounds, int *degenerate) {
  double lo, hi;
  if (mode == 0) {
    double *work = (double *)malloc((size_t)n * sizeof(double));
    if (!work) return -2;
    for (int64_t i = 0; i < n; ++i) work[i] = (double)l[i];
    const double q_lo = 1.0 / 100.0, q_hi = 99.0 / 100.0;
    lo = percentile_linear(work, n, q_lo);
    hi = percentile_linear(work, n, q_hi);
    free(work);
  } else if (mode == 1) {
    if (!(fixed_bound > 0)) return -1;
    lo = -fixed_bound;
    hi = fixed_bound;
  } else {
    return -1;
  }
  bounds[0] = lo;
  bounds[1] = hi;
  if (!(hi > lo)) {
    *degenerate = 1;
    memset(out, 128, (size_t)n);
    return 0;
  }
  *degenerate = 0;
  const double scale = 255.0 / (hi - lo);
  for (int64_t i = 0; i < n; ++i) {
    double s = ((double)l[i] - lo) * scale;
    double r = floor(s + 0.5);
    if (r < 0.0) r = 0.0;
    if (r > 255.0) r = 255.0;
    out[i] = (uint8_t)r;
  }
  return 0;
}

/* EVF1 record block decode (event_io.py:60-76).  Returns -1 when every
 * record is in bounds, else the index of the first out-of-bounds record
 * (outputs are then unspecified; the caller raises DataError). */
int64_t oracle_decode_evf1(const uint8_t *raw, int64_t nrec, int64_t width,
                           int64_t height, uint64_t t_base, uint64_t *t,
                           uint16_t *x, uint16_t *y, int8_t *p) {
  uint64_t acc = 0;
  for (int64_t r = 0; r < nrec; ++r) {
    const uint8_t *rec = raw + 8 * r;
    uint32_t dt = (uint32_t)rec[0] | ((uint32_t)rec[1] << 8) |
                  ((uint32_t)rec[2] << 16) | ((uint32_t)rec[3] << 24);
    uint16_t xp = (uint16_t)(rec[4] | (rec[5] << 8));
    uint16_t yy = (uint16_t)(rec[6] | (rec[7] << 8));
    uint16_t xx = xp & 0x7FFF;
    if (xx >= width || yy >= height) return r;
    acc += dt;
    t[r] = acc + t_base;
    x[r] = xx;
    y[r] = yy;
    p[r] = (xp >> 15) ? 1 : -1;
  }
  return -1;
}

/* Single-pixel two-stage trajectory (_kernels.py:219-233), float32 and float64
 * state; state[0] = p_bar, state[1] = l, updated in place. */
#define ORACLE_TRACE(NAME, T)                                                    \
  void NAME(const int8_t *ps, int64_t n, T a, T oma, T b, T h, T *state,        \
            T *out_pbar, T *out_delta, T *out_l) {                              \
    T pb = state[0], lv = state[1];                                             \
    for (int64_t j = 0; j < n; ++j) {                                           \
      T p = (T)ps[j];                                                           \
      T t1 = a * pb;                                                            \
      T t2 = oma * p;                                                           \
      pb = t1 + t2;                                                             \
      T d = p - pb;                                                             \
      T t3 = b * lv;                                                            \
      T t4 = h * d;                                                             \
      lv = t3 + t4;                                                             \
      out_pbar[j] = pb;                                                         \
      out_delta[j] = d;                                                         \
      out_l[j] = lv;                                                            \
    }                                                                           \
    state[0] = pb;                                                              \
    state[1] = lv;                                                              \
  }
ORACLE_TRACE(oracle_trace_f32, float)
ORACLE_TRACE(oracle_trace_f64, double)

/* Combined recurrence (_kernels.py:236-249): state = (l_prev, l_prev2, p_prev). */
#define ORACLE_TRACE_IIR(NAME, T)                                                \
  void NAME(const int8_t *ps, int64_t n, T apb, T atb, T h, T *state, T *out_l) { \
    T l1 = state[0], l2 = state[1], pp = state[2];                              \
    for (int64_t j = 0; j < n; ++j) {                                           \
      T p = (T)ps[j];                                                           \
      T t1 = apb * l1;                                                          \
      T t2 = atb * l2;                                                          \
      T t3 = t1 - t2;                                                           \
      T t4 = p - pp;                                                            \
      T t5 = h * t4;                                                            \
      T lv = t3 + t5;                                                           \
      out_l[j] = lv;                                                            \
      l2 = l1;                                                                  \
      l1 = lv;                                                                  \
      pp = p;                                                                   \
    }                                                                           \
    state[0] = l1;                                                              \
    state[1] = l2;                                                              \
    state[2] = pp;                                                              \
  }
ORACLE_TRACE_IIR(oracle_trace_iir_f32, float)
ORACLE_TRACE_IIR(oracle_trace_iir_f64, double)

/* Per-pixel ON/OFF counts (calib.py:26-45); returns the first event index
 * whose flat index y*W + x is >= n_pix (counts untouched then), else -1. */
int64_t oracle_count_events(const uint16_t *xs, const uint16_t *ys, const int8_t *ps, int64_t n, int64_t width,
                            int64_t n_pix, int64_t *n_on, int64_t *n_off) {
  for (int64_t e = 0; e < n; ++e)
    if ((int64_t)ys[e] * width + xs[e] >= n_pix) return e;
  for (int64_t e = 0; e < n; ++e) {
    const int64_t f = (int64_t)ys[e] * width + xs[e];
    if (ps[e] > 0) ++n_on[f]; else ++n_off[f];
  }
  return -1;
}
