// fibar_kernels.cuh -- what the engine's translation units share: constants,
// the per-launch context (Ctx), small device helpers and the kernel
// declarations (definitions: fibar_front.cu, fibar_stage.cu, fibar_readout.cu).
#pragma once
#include <cstdint>
#include "fibar_common.cuh"
#include "fibar_internal.h"
#include "../../include/fibar_b200.h"

namespace fibar {

constexpr int NFINE = 10;     // fine candidate windows around the interpolated fixed point
constexpr int CHUNK_MIN = 32;  // smallest speculative window chunk (sizes the chunk arrays)
constexpr int NLIN = 7;      // coarse candidates q0 + c_lin_off[i]
constexpr int NGEO = 12;     // coarse candidates q0 * c_geo_mul[i]
constexpr int NCAND = NLIN + NGEO;
constexpr int TPB = 256;
#ifndef FIBAR_BLUR_MINB
#define FIBAR_BLUR_MINB 1
#endif
constexpr int BLUR_MINB = FIBAR_BLUR_MINB;   // k_blur: min resident blocks per SM (register cap)
#ifndef FIBAR_PREP_MINB
#define FIBAR_PREP_MINB 4
#endif
constexpr int PREP_MINB = FIBAR_PREP_MINB;   // k_blur_prep: min resident blocks per SM
constexpr unsigned ITEM_CARRIED_ONLY = 1u;   // Item.pad flag
constexpr int IN_ITEMS = 8;
constexpr int IN_TILE = TPB * IN_ITEMS;
constexpr unsigned WIN_SOLO = 384;   // evictions a lane counts alone (longer: the whole warp)
constexpr int GROUP = 8;
#ifndef FIBAR_LONG_SEG
#define FIBAR_LONG_SEG 64
#endif
constexpr int LONG_SEG = FIBAR_LONG_SEG;    // segments longer than this go to k_temporal_long
constexpr int LONG_TPB = 256;      // lanes per long segment (one block)
constexpr int LONG_PIECE = 64;     // minimum events per lane before more lanes join
constexpr int EV_PER_THREAD = 2;
constexpr int EV_TILE = TPB * EV_PER_THREAD;
// halo bands: a prep record with this okm is an injected item (val[0] = its in-word slot)
constexpr unsigned HALO_OKM = 1u << 9;
constexpr unsigned TAINT_HI = 0x80000000u;   // taint bit of a value word's high half (bit 63)

// a chunk the window verifier re-runs, with its predecessor's end state as
// read before the round writes anything
struct VRec {
  long long s, q, np, nt, ev;
  int c, pad;
};
#ifndef FIBAR_VF_TPB
#define FIBAR_VF_TPB 256
#endif
constexpr int VF_TPB = FIBAR_VF_TPB;   // k_window_verify: threads per CTA (one warp per re-run)
constexpr int VF_CTAS = 16;   // k_window_verify: CTAs in its one cluster (non-portable size)

// device packets gathered into the device staging set (non-contiguous
// packets coalesced into one batch): the table travels as a kernel parameter
constexpr int GATHER_MAX = 256;
struct GatherEntry {
  const uint16_t *x, *y;
  const int8_t *p;
  long long n, dst;
};
struct GatherTable {
  int n;
  GatherEntry e[GATHER_MAX];
};

struct ChunkRec {
  long long st_s, st_q;                          // state after event b_c - 1 (speculative start)
  long long en_s, en_q, en_np, en_nt, en_ev;     // state after the chunk's last event
  long long qlo, qhi;                            // extrema of the targets set inside the chunk
};

// read-out scratch (k_readout): the bounds first (copied to the host as
// {lo, hi, degenerate}), the grid barrier, what the last CTA publishes, and two
// sets of radix histograms (one per launch parity: a launch clears the set the
// next one uses)
struct alignas(16) SelCounters {
  unsigned hist[3][4][2048];      // [pass][target][digit]
};
struct SelState {
  double lo, hi;
  int degenerate;
  unsigned parity;
  unsigned bar_count, bar_gen;
  unsigned pad0[2];
  alignas(16) unsigned bc[12];    // published by the last CTA: prefixes, residual ranks
  unsigned long long ts[16];      // FIBAR_RO_TIMES: CTA 0's phase stamps
  SelCounters cur[2];
};
constexpr int RO_TPB = 512;                  // k_readout: threads per CTA (one CTA per SM)
constexpr long long RO_SMEM_MAX = 160 << 10;  // slice keys kept on chip up to this many bytes

struct Ctx {
  int W, H, ts, tiles_x, A;
  unsigned band_y0, full_H;   // row band [band_y0, band_y0 + H) of a full_H-row sensor
  long long n_pix;
  long long num, den, qmin, qmax, every;
  long long numA;   // num * A (tile area)
  int reg32x;       // regulate32x applies (numA, den < 2^24, q_max < 2^22, den * q_max < 2^29)
  float alpha, oma, beta, h;
  int use_gain, blur_on, spatial;
  DevState *st;
  BatchState *bs;     // this batch's scalars (parity buffer)
  BatchState *bsn;    // the next batch's (its anchors' predicted start state is written here)
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
  long long n_raw;                // raw events (an upper bound when n_raw_dev is set)
  const long long *n_raw_dev;     // the batch's raw event count in device memory, or null
  unsigned *blockcnt;
  unsigned *ekey;
  int8_t *epol, *spol;
  uint2 *longseg;
  unsigned max_long;              // entries of longseg: batch capacity / LONG_SEG + 1 (every long segment fits)
  unsigned *tkey;                 // unsorted tile-major keys (sort input)
  const unsigned *skey, *sidx;    // sorted keys / batch-local event index
  uint2 *dp;
  unsigned *S;
  unsigned *Qt;     // per batch event: the window target after it (k_window_run / k_window_verify)
  unsigned *pmap;   // per eviction: the batch-relative event that pops it (k_popj_map)
  Item *item;
  PosRec *posrec;
  float *t2;
  unsigned long long *bv64, *mv64;   // (epoch << 32 | float bits) per blur item / per sorted position
  BlurPrep *prep;
  unsigned *colist;           // carried-only stale items (pixels without events in the batch)
  // halo band (filter-ON row band); halo == 0: the whole sensor
  int halo;
  int hreg0, hreg1;          // rows whose blur items this engine takes
  int hin_top, hin_bot;      // rows whose items are injected from the neighbours (-1: none)
  int hout_top, hout_bot;    // rows whose items the neighbours inject (-1: none)
  unsigned *hslot;           // per injected item: its in-word slot
  const unsigned long long *hin;   // this round's in-words
  int chunk, warm, debug;
  int fp_fused;               // k_anchor2 computes the chunks' fixed points itself (small batches)
  int twarm;                  // warm-up events of a speculative long-segment piece
  unsigned blur_sleep;
  unsigned long long *dbg_t, *dbg_g;
  int2 *anc, *anc2;
  int2 *anc0;   // per chunk: distinct counts of the no-pop window [s_start, a_c - 1]
  long long *lc, *lu;
  ChunkRec *ch;
  VRec *vl;
};

struct BatchScalars {
  long long E0, B, s_start, s_end;
  unsigned epoch, epoch0;
};

__device__ __forceinline__ BatchScalars load_bs(const Ctx &x) {
  BatchScalars b;
  b.E0 = x.bs->E0;
  b.B = x.bs->B;
  b.s_start = x.bs->s_start;
  b.s_end = b.s_start + x.bs->npop;
  b.epoch = x.bs->epoch;
  b.epoch0 = x.bs->epoch0;
  return b;
}

__device__ __forceinline__ unsigned order_key(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float order_unkey(unsigned k) {
  const unsigned u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(u);
}

// kernels (launched by fibar_engine.cu)
__global__ void __launch_bounds__(TPB) k_snap(const float *__restrict__ src, float *__restrict__ dst, long long n);
__global__ void __launch_bounds__(TPB) k_debug_regulate(Ctx x, const unsigned *len, const unsigned *np, const unsigned *nt,
                                                        long long n, unsigned *out_fast, unsigned *out_exact);
__global__ void __launch_bounds__(TPB) k_count_inb(Ctx x, int nblocks);
__global__ void __launch_bounds__(TPB) k_compact(Ctx x, int nblocks, int fused);
__global__ void k_batch_begin(Ctx x);
__global__ void k_ingest_end(Ctx x);
__global__ void k_predict(Ctx x);
__global__ void __launch_bounds__(TPB) k_fp(Ctx x);
__global__ void __launch_bounds__(TPB) k_stage(const uint16_t *sx, const uint16_t *sy, const int8_t *sp, long long n,
                                               uint16_t *dx, uint16_t *dy, int8_t *dp, long long *n_dev);
__global__ void __launch_bounds__(TPB) k_gather(const GatherTable tab, uint16_t *dx, uint16_t *dy, int8_t *dp);
__global__ void __launch_bounds__(TPB) k_seg_marks(Ctx x);
__global__ void __launch_bounds__(TPB) k_link(Ctx x);
__global__ void __launch_bounds__(TPB) k_anchor(Ctx x);
__global__ void __launch_bounds__(TPB) k_anchor_base(Ctx x);
__global__ void __launch_bounds__(1024) k_anchor_scan(Ctx x, int2 *anc, int nc);
__global__ void __launch_bounds__(TPB) k_anchor2(Ctx x);
__global__ void __launch_bounds__(128) k_window_run(Ctx x);
__global__ void __launch_bounds__(128) k_window_run_g2(Ctx x);
__global__ void __launch_bounds__(128) k_window_run_g4(Ctx x);
__global__ void __launch_bounds__(128) k_window_run_g8(Ctx x);
__global__ void __launch_bounds__(VF_TPB, VF_TPB > 256 ? 1 : 2) k_window_verify(Ctx x);
__global__ void __launch_bounds__(TPB) k_popj_map(Ctx x);
__global__ void __launch_bounds__(TPB) k_popj(Ctx x);
__global__ void __launch_bounds__(TPB) k_posinfo(Ctx x, int close);
__global__ void __launch_bounds__(TPB) k_temporal(Ctx x);
__global__ void __launch_bounds__(TPB) k_temporal_runs(Ctx x);
__global__ void __launch_bounds__(LONG_TPB) k_temporal_long(Ctx x);
__global__ void __launch_bounds__(TPB, PREP_MINB) k_blur_prep(Ctx x);
__global__ void __launch_bounds__(TPB, BLUR_MINB) k_blur(Ctx x);
__global__ void __launch_bounds__(TPB) k_blur_halo(Ctx x);   // halo-band engines
__global__ void __launch_bounds__(TPB) k_final(Ctx x);
__global__ void k_batch_end(Ctx x);
__global__ void __launch_bounds__(TPB) k_halo_count(Ctx x, unsigned *cnt, int nb);
__global__ void __launch_bounds__(TPB) k_halo_write(Ctx x, const unsigned *cnt, int nb, unsigned *hlist);
__global__ void k_halo_epoch(Ctx x);
__global__ void __launch_bounds__(TPB) k_halo_collect(Ctx x, const unsigned *hlist, long long n_in, long long n_out,
                                                      unsigned long long *out);
#ifndef FIBAR_RO_MINB
#define FIBAR_RO_MINB 2
#endif
__global__ void __launch_bounds__(RO_TPB, FIBAR_RO_MINB) k_readout(const float *__restrict__ l, long long n, SelState *sel, int mode, double fixed_bound, uint4 ranks, double g_lo, double g_hi, uint8_t *__restrict__ out, long long slice, int on_chip);
__global__ void __launch_bounds__(TPB) k_evf1_decode(const uint4 *__restrict__ rec2, const uint2 *__restrict__ rec1, long long nrec, int W, int H, uint16_t *__restrict__ xo, uint16_t *__restrict__ yo, int8_t *__restrict__ po, unsigned *__restrict__ dto, unsigned long long *__restrict__ bsum, unsigned long long *__restrict__ first_bad);
__global__ void __launch_bounds__(1024) k_evf1_block_scan(unsigned long long *bsum, int nb, unsigned long long t_base);
__global__ void __launch_bounds__(TPB) k_evf1_times(const unsigned *__restrict__ dt, long long nrec, const unsigned long long *__restrict__ bofs, unsigned long long *__restrict__ t);
__global__ void k_active_counts(Ctx x, unsigned *cnt);
__global__ void k_tile_counts(Ctx x, const unsigned *cnt, unsigned *tcnt);
__global__ void k_ring_xy(Ctx x, uint16_t *qx, uint16_t *qy);
__global__ void k_init_state(DevState *s, long long q0, BatchState *bs, int nbs);
__global__ void k_fill_ll(long long *p, long long n, long long v);
__global__ void k_init_pt(PixRec *p, long long *plast, long long n);

}  // namespace fibar
