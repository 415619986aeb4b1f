/*
 * fibar_b200.h -- C ABI of the B200-native FIBAR reconstruction hot path.
 *
 * A plain C interface (opaque handle, plain pointers and sizes, no torch types)
 * that replaces the reference's native layer for the event->image path.  Each
 * entry point names the reference interface it stands in for
 * (paths relative to /root/reference/pkg/src/fibar):
 *
 *   fibar_create / fibar_destroy
 *       ReconstructionEngine.__init__ state allocation, pipeline.py:66-124
 *       (p_bar, l, active_count, tile_count, ring qx/qy, qs[10], gain map,
 *       float32 coefficient casts).
 *   fibar_process
 *       ReconstructionEngine.process_array, pipeline.py:196-243, i.e. the OOB
 *       filter (non-strict) plus the numba kernels _temporal_chunk
 *       (_kernels.py:62-73) / _full_chunk (_kernels.py:76-216).
 *   fibar_flush
 *       (no reference equivalent: the engine coalesces packets on the device
 *       between read-outs; state is packet-size invariant).
 *   fibar_render / fibar_render_async
 *       ReconstructionEngine.render, pipeline.py:247-269 (async: the frame
 *       loop of run(), pipeline.py:372-397, without a host wait per frame).
 *   fibar_read_qs / fibar_counters
 *       the qs[10] slots (_kernels.py:48-59, pipeline.py:136-162) and
 *       event_count / oob_dropped (pipeline.py:122-124).
 *   fibar_read_state
 *       the arrays hashed by state_digest / returned by iap, l_grid,
 *       p_bar_grid (pipeline.py:128-181).
 *   fibar_halo_batch / fibar_halo_round / fibar_halo_finish
 *       _full_chunk (_kernels.py:76-216) for one row band of a filter-ON
 *       multi-GPU partition: the window pass of the whole stream, the blur loop
 *       (_kernels.py:173-189) for the band's rows, halo values exchanged by the
 *       caller between rounds.
 *
 * Threading: one engine = one CUDA stream; calls on one engine must not race
 * (same contract as the reference).  Every call returns 0 on
 * success or one of the FIBAR_E_* codes below; the Python shim maps them to
 * the reference's exception classes (errors.py).
 */
#ifndef FIBAR_B200_H
#define FIBAR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FIBAR_OK 0
#define FIBAR_E_CONFIG 1     /* -> ConfigError */
#define FIBAR_E_DATA 2       /* -> DataError */
#define FIBAR_E_ORDER 3      /* -> OrderError */
#define FIBAR_E_INVARIANT 4  /* -> InvariantError (e.g. counter saturation) */
#define FIBAR_E_CUDA 5       /* -> DeviceError */
#define FIBAR_E_NODEVICE 6   /* -> DeviceError */

#define FIBAR_MEM_HOST 0
#define FIBAR_MEM_DEVICE 1

#define FIBAR_RENDER_ROBUST 0
#define FIBAR_RENDER_FIXED 1

typedef struct fibar_engine fibar_engine;

typedef struct fibar_config {
  int32_t width;
  int32_t height;
  int32_t tile_side;        /* FilterParams.tile_side (core.py:68) */
  int32_t spatial_enabled;  /* FilterParams.spatial_enabled (core.py:71) */
  int32_t blur_enabled;     /* ReconstructionEngine(blur_enabled=) */
  int32_t reserved0;
  int64_t regulate_every;   /* ReconstructionEngine(regulate_every=) */
  int64_t fill_num;         /* fill_ratio_target numerator / denominator */
  int64_t fill_den;
  int64_t q_min;
  int64_t q_max;
  float alpha;              /* float32(params.alpha)            pipeline.py:117 */
  float one_m_alpha;        /* float32(1 - params.alpha)        pipeline.py:118 */
  float beta;               /* float32(params.beta)             pipeline.py:119 */
  float half_1p_beta;       /* float32(params.half_one_plus_beta) pipeline.py:120 */
  const float *gain;        /* optional host array [height*width] or NULL */
  int64_t batch_capacity;   /* max in-bounds events per device batch; 0 = default */
  /* Row band (multi-GPU row-band partition, filter OFF only): this engine owns
   * rows [band_y0, band_y0 + height) of a sensor_height-row sensor; events of
   * other rows are left to their band's owner.  sensor_height = 0: no band. */
  int32_t band_y0;
  int32_t sensor_height;
  /* Halo band (multi-GPU row-band partition, filter ON): the
   * engine keeps the whole sensor's window (every rank sees every event) but
   * blurs only the items of rows [halo_own_y0 - halo_rows, halo_own_y1 +
   * halo_rows); the outermost of those rows, when it belongs to a neighbour,
   * takes its blurred values from that neighbour (fibar_halo_round).
   * halo_own_y1 = 0: off. */
  int32_t halo_own_y0;
  int32_t halo_own_y1;
  int32_t halo_rows;
  int32_t reserved1;
} fibar_config;

/* Allocate device state for one sensor.  stream: a cudaStream_t (NULL = legacy default). */
int fibar_create(const fibar_config *cfg, void *stream, fibar_engine **out);
int fibar_destroy(fibar_engine *eng);
int fibar_set_stream(fibar_engine *eng, void *stream);
/* Return to the freshly constructed state (zero filter state, empty window). */
int fibar_reset(fibar_engine *eng);

/* Append one packet of n events (SoA columns x, y uint16 and p int8 in {-1,+1}).
 * mem = FIBAR_MEM_HOST or FIBAR_MEM_DEVICE says where the three columns live.
 * Out-of-bounds events are dropped and counted (non-strict semantics of
 * pipeline.py:201-213); strict checks are the caller's.  Work is queued on the
 * engine stream; packets may be coalesced until the next read. */
int fibar_process(fibar_engine *eng, const uint16_t *x, const uint16_t *y, const int8_t *p, int64_t n,
                  int32_t mem);
/* Run any coalesced events now (asynchronous on the engine stream). */
int fibar_flush(fibar_engine *eng);
/* Events waiting for the next batch: device_events are read in place from the
 * caller's device buffers (contiguous device packets are coalesced without a
 * copy), so those buffers must stay valid until this count drops to 0. */
int fibar_pending(fibar_engine *eng, int64_t *device_events, int64_t *staged_events);

/* Render the brightness grid to uint8 [height*width].  out_mem says where
 * `out` lives.  bounds (host double[2]) and degenerate (host int) are written
 * after a stream synchronisation; pass NULL to skip them (then nothing blocks
 * when out is device memory). */
int fibar_render(fibar_engine *eng, int32_t mode, double fixed_bound, uint8_t *out, int32_t out_mem,
                 double *bounds, int32_t *degenerate);

/* Asynchronous read-out (pipeline.run's frame loop): the same frame as
 * fibar_render, enqueued after the newest blur stage on the engine's blur
 * stream so the next batch's front end overlaps it.  Nothing blocks and the
 * caller's stream does not wait: `ready` (a cudaEvent_t made by the caller) is
 * recorded when out (uint8 [n_pix], device or pinned host per out_mem) and
 * meta (same memory kind: double lo, double hi, int32 degenerate) are
 * written.  Later batches order after the read-out. */
int fibar_render_async(fibar_engine *eng, int32_t mode, double fixed_bound, uint8_t *out, int32_t out_mem, void *meta,
                       void *ready);

/* Synchronising reads (host pointers). */
int fibar_read_qs(fibar_engine *eng, int64_t qs[10]);
int fibar_counters(fibar_engine *eng, int64_t *event_count, int64_t *oob_dropped);
/* Any pointer may be NULL.  Sizes: p_bar, l: n_pix float; active: n_pix uint16;
 * tiles: tiles_x*tiles_y uint8; qx, qy: n_pix+1 uint16. */
int fibar_read_state(fibar_engine *eng, float *p_bar, float *l, uint16_t *active, uint8_t *tiles,
                     uint16_t *qx, uint16_t *qy);

/* Parity surface for the stale mask (runs pending packets first): the stale
 * episodes of the most recent device batch, in pop order -- the in-bounds
 * index of the event whose trim made the pixel stale and the pixel (row-major,
 * engine rows) -- i.e. the per-event blurred-pixel list of the reference's
 * SpatialFilter.on_event (spatial.py:165-207) / the stale branch of
 * _kernels.py:160-172 for that batch.  *n_out = the count; fails if it
 * exceeds cap.  Filter ON only (else *n_out = 0). */
int fibar_debug_stale_items(fibar_engine *eng, int64_t *event_idx, uint32_t *pixel, int64_t cap, int64_t *n_out);

/* Parity surface for the window regulator: the 32-bit form the window kernels
 * use (float quotient + exact remainder fix-up) beside the reference's integer
 * formula q = clamp(len * n_tiles * A * num // (den * n_pix), q_min, q_max)
 * (_kernels.py:195-201) in exact 64-bit arithmetic, for n host triples
 * (len, n_pix_active, n_tiles_active), n_pix_active >= 1.  Fails unless the
 * 32-bit form applies (num * A, den < 2^24, q_max < 2^22, den * q_max < 2^29). */
int fibar_debug_regulate(int64_t num, int64_t den, int32_t tile_area, int64_t q_min, int64_t q_max, const uint32_t *len,
                         const uint32_t *np, const uint32_t *nt, int64_t n, uint32_t *out_fast, uint32_t *out_exact);

/* Measurement: with FIBAR_TRACE=1 set at creation, timing events are recorded
 * at the stream-part boundaries of every streamed batch (labels 0/1 ingest
 * start/end, 2/3 window part, 4/5 eviction pass, 6/7 blur stage, 8 read-out
 * end).  Returns (batch index, label, ms since the first mark) and clears them;
 * synchronises the device. */
int fibar_debug_trace(fibar_engine *eng, int64_t cap, int64_t *batch, int32_t *label, double *ms, int64_t *n_out);

/* Diagnostics (runs pending packets first): stats[0] = device kernel launches
 * so far, [1] = device batches, [2] = speculative window chunks, [3] = chunks
 * re-run by the verifier, [4] = pops (window evictions) processed, [5] =
 * counter-saturation flag (> 0 once the reference's u16
 * active_count -- or u8 tile_count when a tile has > 255 pixels -- could have
 * hit its cap; conservative, never missed), [6] = in-bounds events, [7] =
 * batch capacity, [8] = evictions replayed in speculative warm-ups, [9] =
 * warp-cooperative eviction-count steps, [10] = window verifier rounds, [11] =
 * FIBAR_DEBUG_WINDOW anchor recount mismatches. */
int fibar_stats(fibar_engine *eng, int64_t stats[16]);
/* Per-kernel CUDA-event timing (bench.py's roofline leg; adds events around
 * every launch, so never enable it in a timed region).  fibar_profile
 * synchronises and clears; fibar_profile_read aggregates by kernel name:
 * names is max_entries x name_len chars, total_ms / launches per entry. */
int fibar_profile(fibar_engine *eng, int32_t enable);
int fibar_profile_read(fibar_engine *eng, int32_t max_entries, char *names, int32_t name_len, double *total_ms,
                       int64_t *launches, int32_t *n_entries);
/* Debug only (env FIBAR_DEBUG_TIMES at create): blur item completion and
 * take-up timestamps (ns, %globaltimer) of the last batch, n items. */
int fibar_debug_times(fibar_engine *eng, uint64_t *done_ns, uint64_t *grab_ns, int64_t n);
/* Debug only: the blur items' resolved-tap records of the last batch (80 B each). */
int fibar_debug_prep(fibar_engine *eng, void *out, int64_t n);
/* debug: globaltimer stamps (ns) of the last read-out's phases, CTA 0
 * (16 slots; zero unless the library was built with FIBAR_RO_TIMES) */
int fibar_debug_readout_times(fibar_engine *eng, uint64_t ts[16]);
/* Copy the float32 brightness grid (after running coalesced events) to dst
 * (dst_mem: FIBAR_MEM_DEVICE, asynchronous; or FIBAR_MEM_HOST, synchronous). */
int fibar_copy_brightness(fibar_engine *eng, float *dst, int32_t dst_mem);
/* Device pointer of the float32 brightness grid (valid until destroy). */
int fibar_brightness_ptr(fibar_engine *eng, float **out);

/* Stateless read-out of any device float32 grid of n pixels (e.g. a full frame
 * assembled from row bands), same semantics as fibar_render.  stream: cudaStream_t. */
int fibar_render_grid(const float *l_dev, int64_t n, int32_t mode, double fixed_bound, uint8_t *out,
                      int32_t out_mem, double *bounds, int32_t *degenerate, void *stream);

/* Decode nrec EVF1 records (event_io.py:60-76: dt u32 | xp u16 | y u16,
 * little endian) already in device memory into device columns x, y (uint16),
 * p (int8 +-1) and, if t is non-NULL, t = t_base + cumulative dt (uint64).
 * records must be 16-byte aligned.  *first_bad receives the index of the
 * first record outside width x height, or -1 (the caller raises DataError as
 * the reference's decoder does).  Synchronises the stream. */
int fibar_decode_evf1(const uint8_t *records, int64_t nrec, int32_t width, int32_t height, uint64_t t_base,
                      uint16_t *x, uint16_t *y, int8_t *p, uint64_t *t, int64_t *first_bad, void *stream);

/* Per-pixel ON / OFF event counts, calib.count_events (calib.py:26-45): for
 * each event flat = y*width + x (as the reference forms it); counts are ADDED
 * into the device int64 arrays n_on / n_off (n_pix each; zero them first).
 * *first_bad receives the index of the first event with flat >= n_pix, or -1
 * (the caller raises DataError like the reference).  x, y, p are device
 * pointers.  Synchronises the stream. */
int fibar_count_events(const uint16_t *x, const uint16_t *y, const int8_t *p, int64_t n, int32_t width, int64_t n_pix,
                       int64_t *n_on, int64_t *n_off, int64_t *first_bad, void *stream);

/* Single-pixel trajectories, temporal.stream_pixel -> _kernels.temporal_trace
 * (_kernels.py:219-233): ntraces independent polarity sequences of n int8
 * values each (trace i at p + i*n), dtype 0 = float32 / 1 = float64 state;
 * coef = {alpha, 1-alpha, beta, (1+beta)/2} as float64, cast to dtype;
 * state = 2 values per trace (p_bar, l) read and updated; p_bar / delta / l
 * receive n values per trace.  All pointers are device pointers; asynchronous. */
int fibar_pixel_trace(const int8_t *p, int64_t n, int32_t ntraces, int32_t dtype, const double coef[4], void *state,
                      void *p_bar, void *delta, void *l, void *stream);
/* The combined recurrence, temporal.stream_pixel_iir -> _kernels.iir_trace
 * (_kernels.py:236-249): coef = {alpha+beta, alpha*beta, alpha*(1+beta)/2};
 * state = 3 values per trace (l_prev, l_prev2, p_prev). */
int fibar_pixel_trace_iir(const int8_t *p, int64_t n, int32_t ntraces, int32_t dtype, const double coef[3],
                          void *state, void *l, void *stream);

/* Halo-band batches (engines created with halo_own_y1 > 0).  The host drives
 * one batch at a time through rounds of halo exchange:
 *
 *   fibar_halo_batch   ingest, window pass, stale items, temporal replay and
 *                      blur-tap resolution of one batch of n <= batch_capacity
 *                      events (mem: where x/y/p live); synchronises and returns
 *                      counts = {in_top, in_bot, out_top, out_bot}: the blur
 *                      items of the injected rows (values to receive from the
 *                      neighbours above / below) and of the rows those
 *                      neighbours inject (values to send).  Both sides derive
 *                      the same lists from the same global window, in pop order.
 *   fibar_halo_round   one blur round (asynchronous).  in: in_top + in_bot
 *                      words from the neighbours' last round, out: out_top +
 *                      out_bot words.  A word is (bit 63: tainted | float bits
 *                      in bits 0-31); tainted = the value depends on a halo
 *                      value that was not yet final.  round 0 must pass all
 *                      in-words tainted; later rounds recompute only items
 *                      that were tainted.  When every rank's in-words of a
 *                      round were untainted, that round was exact everywhere.
 *   fibar_halo_finish  end-of-batch brightness (after the last round).
 *
 * These replace the blur loop of _full_chunk (_kernels.py:173-189) for a row
 * band; the window pass is the same as fibar_process's. */
int fibar_halo_batch(fibar_engine *eng, const uint16_t *x, const uint16_t *y, const int8_t *p, int64_t n, int32_t mem,
                     int64_t counts[4]);
int fibar_halo_round(fibar_engine *eng, int32_t round, const uint64_t *in_words, uint64_t *out_words);
int fibar_halo_finish(fibar_engine *eng);

const char *fibar_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FIBAR_B200_H */
