// fibar_common.cuh -- shared device types and helpers for the FIBAR sm_100a path.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define FIBAR_INF32 0xFFFFFFFFu

// Per-pixel batch record (16 B, one load per pixel touch), one table per batch
// parity so batch k+1's front end can run while batch k's blur reads its own.
// (The pixel's last event index before the batch -- the reference's implicit
// "is the pixel still queued" history -- lives in a separate last-touch array.)
//   st/end : [st, end) positions of the pixel's events in the current batch's
//          pixel-sorted order (st == end: no events this batch).  Reset by the
//          final pass, so the table is clean at every batch start.
//   carried : blur item of the pixel's `last` event when that event is evicted
//          stale during the current batch (else FIBAR_NONE); reset by the final pass.
struct __align__(16) PixRec {
  unsigned st;
  unsigned end;
  unsigned carried;
  unsigned pad0;
};

#define FIBAR_NONE 0xFFFFFFFFu

// Per sorted position of the current batch (16 B, one load per tap):
//   jj      : batch-local event index (stream order)
//   bidx    : blur item of this event if it is evicted stale in this batch, else NONE
//   runbase : blur item whose value this position's brightness is built on
//             (latest earlier blur of the same pixel in the batch), else NONE
//   val     : brightness right after this event's temporal update; written by
//             the temporal pass when runbase == NONE, else by blur item runbase
struct __align__(16) PosRec {
  unsigned jj;
  unsigned bidx;
  unsigned runbase;
  float val;
};

// Per eviction item (popped window entry) of the current batch.
struct __align__(16) Item {
  unsigned jrel;    // batch-local index of the event whose trim popped it
  unsigned pix;     // pixel (row-major) if the entry went stale, else NONE
  unsigned runpos;  // first sorted position whose brightness builds on this blur, else NONE
  unsigned pad;
};

// A blur item's taps after the dependency-free part of their resolution
// (48 B, three 16-byte loads): tap t is in bounds iff bit t of okm; pending
// iff bit t of pend, in which case val[t] names the word to wait for (bit 31:
// a rebuilt-run position, else a blur item); otherwise val[t] holds the float
// bits of the tap's brightness.  runpos: the item's first rebuilt position.
struct __align__(16) BlurPrep {
  unsigned okm, pend;
  unsigned val[9];
  unsigned runpos;
};

// Scalars of one device batch (double buffered by batch parity).
struct BatchState {
  long long E0;        // in-bounds events before the batch (global index of its first event)
  long long B;         // in-bounds events of the batch
  long long s_start;   // window start when the batch began
  long long npop;      // evictions of the batch (set by the window verifier)
  long long stale_batch;
  unsigned epoch;      // batch counter (tags blur words)
  unsigned ticket;     // blur work ticket
  unsigned nlong;      // long pixel segments
  unsigned nco;        // stale items of pixels with no events in the batch (listed by k_popj)
  unsigned epoch0;     // the batch's first epoch (halo bands: one more per exchange round)
  unsigned nbad;       // (unused)
  long long qlo, qhi;  // extrema of the targets set in the batch (k_window_verify)
  unsigned vcnt[3];    // k_window_verify: chunks listed for a round (rotating by round)
  unsigned vpad;
  long long n_raw;     // raw events of the batch, set by k_stage (graphs are captured per size class)
  unsigned nclosed;    // k_posinfo blocks done (the last one closes the batch)
  int geo_next;        // (unused)
  // The state the batch's anchors count their candidate windows against: a
  // predicted window at the batch start with exact distinct counts, written by
  // the previous batch's anchors (k_predict) -- so anchors never wait for the
  // previous window run or verifier.  p_geo: add the geometric candidates.
  int p_geo;
  long long p_s, p_q, p_np, p_nt;
  long long s_anchor;  // p_s as the batch's anchors used it (k_window_run reads this copy)
};

// Window / counter state living in device memory so no kernel needs a host
// round trip.  Mirrors the reference's qs[10] slots (_kernels.py:48-59) plus
// the engine counters (pipeline.py:122-124).
struct DevState {
  long long s;        // window start (global in-bounds index); QS_HEAD = s mod (n_pix+1)
  long long q;        // QS_TARGET
  long long npix;     // QS_NPIX
  long long ntiles;   // QS_NTILES
  long long evctr;    // QS_EVCTR
  long long qtmin;    // QS_QTMIN
  long long qtmax;    // QS_QTMAX
  long long blur;     // QS_BLUR
  long long stale;    // QS_STALE
  long long E;        // in-bounds events consumed (event_count)
  long long oob;      // oob_dropped
  long long B;        // in-bounds events of the batch being processed
  long long s_start;  // window start when the batch began
  long long chunks;   // speculative window chunks launched (stats)
  long long mismatch; // chunks re-run by the verifier (stats)
  long long pops;     // total evictions (stats)
  long long stale_batch;
  long long npop;      // evictions of the batch being processed (set by the window verifier)
  unsigned epoch;     // batch counter (tags blur ready flags)
  unsigned ticket;    // blur work ticket
  unsigned qhead, qtail, qtail_res, qpad;   // blur ready FIFO
  unsigned long long blur_done;              // blur items finished in this batch
  long long saturated;
  long long warm_pops;   // evictions replayed during speculative warm-ups (stats)
  long long coop_iters;  // warp-cooperative eviction-count steps (stats)
  long long fix_rounds;  // verifier rounds (stats)
  int geo, geo_unused;   // window candidates: geometric set needed (set by the previous batch's verifier)
  unsigned nlong, nlong_pad;   // long pixel segments of the batch
  long long dbg_bad;           // FIBAR_DEBUG_WINDOW: anchor counts that disagreed with a serial recount
  long long Ein;               // in-bounds events ingested (the ingest's running E, ahead of E)

};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel_u32(unsigned *p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u32(unsigned *p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// strictly IEEE, separately rounded float32 arithmetic (no FMA contraction),
// matching the reference's numba kernels bit for bit.
__device__ __forceinline__ float fmulr(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float faddr(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsubr(float a, float b) { return __fsub_rn(a, b); }

__device__ __forceinline__ unsigned dist32(long long later, long long earlier) {
  long long d = later - earlier;
  return (earlier < 0 || d >= (long long)FIBAR_INF32) ? FIBAR_INF32 : (unsigned)d;
}
