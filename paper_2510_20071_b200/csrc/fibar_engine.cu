// fibar_engine.cu -- B200-native FIBAR reconstruction engine (sm_100a): engine
// state, batch orchestration (streams, events, graphs) and the C ABI.  Kernels
// live in fibar_front.cu (ingest / link / window / stale), fibar_stage.cu
// (temporal / blur / final), fibar_readout.cu (read-out, EVF1, state export) and
// fibar_sort.cu (radix sort, scans); fibar_kernels.cuh declares them.
//
// One device batch (coalesced packets) flows through:
//   ingest     k_count_inb / k_compact      OOB filter + compaction (pipeline.py:201-213),
//                                            pixel keys, ring of window keys
//   group      radix_sort_pairs              stable (tile-major key, index) sort
//   link       k_seg_marks / k_link          per event: distance to previous same-pixel /
//                                            same-tile event; per ring slot: distance to next
//   window     k_anchor / k_anchor_scan /    the reference's FIFO window (_kernels.py:132-205)
//              k_fp / k_anchor2 /            reproduced exactly by chunked speculation +
//              k_window_run_g8 /             verification
//              k_window_verify
//   stale      k_popj                        eviction event of every popped entry; stale iff
//                                            the pixel has no later event before its eviction
//   temporal   k_posinfo / k_temporal_runs / per-pixel in-order replay of the two-stage IIR
//              k_temporal_long               (_kernels.py:62-73 / 120-130), bit exact;
//                                            last-touch tables for the next batch
//   blur       k_blur_prep / k_blur          3x3 renormalised blur of stale pixels in eviction
//                                            order (_kernels.py:173-189), dataflow over a
//                                            persistent grid polling (epoch | value) words
//   final      k_final / k_batch_end         end-of-batch brightness, counters
//   read-out   k_readout                     exact percentile select + float64 map in one
//                                            cooperative kernel (pipeline.py:247-269)
//
// Filter ON, a batch's parts run on the engine's own streams -- sort, links +
// anchors, window, eviction, blur stage, read-out -- with about five batches in
// flight; small batches replay one captured CUDA graph per part
// (4.6); consecutive kernels use programmatic dependent launch (pdl_wait()).
// Float32 arithmetic uses __fmul_rn/__fadd_rn (never contracted to FMA) so the
// result is bit-identical to the reference's strict-IEEE numba kernels.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <algorithm>
#include <chrono>
#include <string>
#include <mutex>
#include <vector>

#include <cuda.h>

#include "fibar_kernels.cuh"

using namespace fibar;

namespace fibar {
thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char *where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return FIBAR_E_CUDA;
}
}  // namespace fibar

namespace {

// CUDA driver entry points for green contexts, resolved at run time through
// the runtime (cudaGetDriverEntryPoint), so the library does not link libcuda
// and still loads where no driver is installed (the CPU build/test host).
struct GreenApi {
  bool ok = false;
  CUresult (*deviceGet)(CUdevice *, int) = nullptr;
  CUresult (*getDevResource)(CUdevice, CUdevResource *, CUdevResourceType) = nullptr;
  CUresult (*splitByCount)(CUdevResource *, unsigned *, const CUdevResource *, CUdevResource *, unsigned,
                           unsigned) = nullptr;
  CUresult (*generateDesc)(CUdevResourceDesc *, CUdevResource *, unsigned) = nullptr;
  CUresult (*ctxCreate)(CUgreenCtx *, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
  CUresult (*streamCreate)(CUstream *, CUgreenCtx, unsigned, int) = nullptr;
  CUresult (*ctxDestroy)(CUgreenCtx) = nullptr;
};

template <class F>
bool driver_fn(const char *name, F &fn) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !p) {
    cudaGetLastError();
    return false;
  }
  fn = reinterpret_cast<F>(p);
  return true;
}

const GreenApi &green_api() {
  static GreenApi api = [] {
    GreenApi a;
    a.ok = driver_fn("cuDeviceGet", a.deviceGet) && driver_fn("cuDeviceGetDevResource", a.getDevResource) &&
           driver_fn("cuDevSmResourceSplitByCount", a.splitByCount) &&
           driver_fn("cuDevResourceGenerateDesc", a.generateDesc) && driver_fn("cuGreenCtxCreate", a.ctxCreate) &&
           driver_fn("cuGreenCtxStreamCreate", a.streamCreate) && driver_fn("cuGreenCtxDestroy", a.ctxDestroy);
    return a;
  }();
  return api;
}

int ceil_log2(long long v) {
  int b = 0;
  while ((1LL << b) < v) ++b;
  return b;
}

}  // namespace

// buffer sets for batches in flight (ingest of k+2 may run while k's window
// part and k-1's blur stage run), indexed by batch % NPAR
#ifndef FIBAR_NPAR
#define FIBAR_NPAR 5
#endif
constexpr int NPAR = FIBAR_NPAR;

// small batches' front-end graphs are captured per size class of this many events
constexpr long long GRAPH_CLASS = 16384;

struct GraphEntry {
  long long n;               // batch size the graph was captured for
  long long kernels;         // kernels per replay (the launch counter)
  cudaGraphExec_t exec = nullptr;
  cudaGraphExec_t exec2 = nullptr;   // kind 1: the window part (exec: the ingest)
  long long kernels2 = 0;
  cudaGraphExec_t exec3 = nullptr;   // kind 1: the eviction pass
  long long kernels3 = 0;
  cudaGraphExec_t exec4 = nullptr;   // kind 1: the anchors (exec2: run + verifier)
  long long kernels4 = 0;
  cudaGraphExec_t exec5 = nullptr;   // kind 1: segments, links and the anchors (exec: the sort part of the ingest)
  long long kernels5 = 0;
  cudaGraphExec_t exec6 = nullptr;   // kind 1: the blur stage (replay, tap resolution, blur dataflow, final)
  long long kernels6 = 0;
  int kind = 0;              // 0: whole batch (serial schedule), 1: front end of the streamed schedule (two parts)
  int par = 0;               // kind 1: the batch parity whose buffers it uses
  int where = 0;             // kind 1: which radix-sort buffer holds the sorted keys
};

struct fibar_engine {
  fibar_config cfg{};
  int W = 0, H = 0, ts = 2, A = 4, tiles_x = 0, tiles_y = 0;
  unsigned band_y0 = 0, full_H = 0;
  long long n_pix = 0, n_tiles = 0;
  long long q0 = 0;
  Launcher L;
  long long Bcap = 0;
  int key_bits = 0;
  long long R = 0;
  bool spatial = true, blur_on = true, use_gain = false;
  DevState *st = nullptr;
  float *pbar = nullptr, *l = nullptr, *gain = nullptr;
  PixRec *pt2[NPAR] = {};
  long long *plast = nullptr;
  unsigned *wcnt = nullptr;
  BatchState *bsd = nullptr;   // [NPAR]
  long long *last_tile = nullptr;
  uint2 *ptt2[NPAR] = {};   // tile segments, per batch parity
  unsigned *rkey = nullptr;
  uint2 *rnext = nullptr;
  uint16_t *raw_x = nullptr, *raw_y = nullptr;
  int8_t *raw_p = nullptr;
  unsigned *blockcnt2[NPAR] = {};   // per buffer set: two batches' sorts may be in flight (astream / astream2)
  unsigned *ekey2[NPAR] = {};
  // polarities in stream order (per batch parity: the next batch's ingest may
  // run while this one's front end reads them) and in pixel-sorted order (per
  // parity: the temporal replay on the blur stream reads them while the next
  // front end writes its own)
  int8_t *epol2[NPAR] = {}, *spol2[NPAR] = {};
  uint2 *longseg2[NPAR] = {};   // long pixel segments, per buffer set (filter ON: listed by the ingest's k_link)
  unsigned *ka2[NPAR] = {}, *va2[NPAR] = {}, *kb2[NPAR] = {}, *vb2[NPAR] = {}, *hist2[NPAR] = {};
  uint2 *dp2[NPAR] = {};    // per-event link distances, per batch parity
  // window starts / targets after each event and the eviction -> popping-event
  // map, per batch parity (the eviction pass of batch k runs beside the window
  // pass of batch k+1)
  unsigned *S2[NPAR] = {}, *Qt2[NPAR] = {}, *pmap2[NPAR] = {};
  unsigned long long *bv64 = nullptr, *mv64 = nullptr;
  BlurPrep *prep = nullptr;            // = prep2[0] (debug reads)
  BlurPrep *prep2[NPAR] = {};   // per batch parity: k_popj of batch k+1 writes while batch k blurs
  // carried-only stale items, per batch parity: k_popj of batch k+2 may run
  // while batch k+1's tap resolution still reads its list
  unsigned *colist2[NPAR] = {};
  Item *item2[NPAR] = {};
  PosRec *posrec2[NPAR] = {};
  float *t2_2[NPAR] = {};
  // window candidates, per buffer set (a batch's anchors run while the
  // previous batch's window run still reads its own)
  int2 *anc3[NPAR] = {}, *anc23[NPAR] = {}, *anc03[NPAR] = {};
  long long *lc3[NPAR] = {}, *lu3[NPAR] = {};
  ChunkRec *ch = nullptr;
  VRec *vl = nullptr;
  SelState *sel = nullptr;
  uint8_t *frame = nullptr;
  unsigned *cnt_tmp = nullptr, *tcnt_tmp = nullptr;
  uint16_t *q_tmp = nullptr;
  // host packets: CPU copy into pinned staging set `cur`, one H2D per batch on
  // a copy stream into device staging set `cur`, double buffered so the copy
  // of batch k+1 overlaps the compute of batch k
  uint16_t *hx[2] = {nullptr, nullptr}, *hy[2] = {nullptr, nullptr};
  int8_t *hp[2] = {nullptr, nullptr};
  uint16_t *sx[2] = {nullptr, nullptr}, *sy[2] = {nullptr, nullptr};
  int8_t *sp_[2] = {nullptr, nullptr};
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  int cur = 0;
  long long hfill = 0;
  const uint16_t *zx = nullptr, *zy = nullptr;  // pending zero-copy device range (contiguous device packets)
  const int8_t *zp = nullptr;
  long long zn = 0;
  // pending non-contiguous device packets, gathered into device staging set
  // `cur` (k_gather) when the batch is full or at a flush point
  GatherTable gt{};
  long long dfill = 0;
  long long batches = 0;
  // filter ON: batch k's blur stage (blur_prep, blur, final) runs on bstream
  // while batch k+1's front end runs on the engine stream; per-batch buffers
  // are double buffered by batch parity
  cudaStream_t bstream = nullptr;
  // FIBAR_GREEN=n: the blur kernel runs in a green context of n SMs
  CUgreenCtx gctx = nullptr;
  cudaStream_t gstream = nullptr;
  cudaEvent_t evP = nullptr, evG = nullptr;
  cudaEvent_t evT = nullptr;   // (unused)
  // streamed filter-ON batches: the front end's ingest + sort (astream) and
  // window part (fstream), so batch k+1's ingest overlaps batch k's window pass
  cudaStream_t astream = nullptr, fstream = nullptr;
  // small batches: the sort part of the ingest alternates between astream and
  // astream2 (it reads nothing of the previous batch); segments and links,
  // which do, follow on lstream in batch order
  cudaStream_t astream2 = nullptr, astream3 = nullptr, lstream = nullptr;
  int sort_lanes = 2;   // FIBAR_SORT_LANES: streams a small batch's sort part rotates over (1..3)
  // asynchronous read-outs: a snapshot of l on the blur stream, the read-out
  // itself on rstream beside the next batch's blur stage
  cudaStream_t rstream = nullptr;
  cudaStream_t tstream = nullptr;   // long-segment replay beside the short segments'
  cudaEvent_t evT0 = nullptr, evT1 = nullptr;
  float *snap[2] = {};
  cudaEvent_t evSnap = nullptr, evRd[2] = {};
  bool rd_used[2] = {};
  long long n_snap = 0;
  bool snap_on = true;   // FIBAR_SNAP=0: the read-out on the blur stream itself
  cudaEvent_t evS[NPAR] = {};   // the set's sort part is done
  cudaEvent_t evIn = nullptr, evCp = nullptr, evA[NPAR] = {};
  // ... and the eviction pass (pstream) after the window part (evV), beside
  // the next batch's window part
  cudaStream_t pstream = nullptr;
  cudaEvent_t evV[NPAR] = {};
  // ... and the anchors (nstream) after the ingest (evA) and the previous
  // batch's run (evR), beside the previous batch's verifier
  cudaStream_t nstream = nullptr;
  cudaEvent_t evN[NPAR] = {}, evR[NPAR] = {};
  int r_par = -1;   // buffer set of the newest batch whose run recorded evR (-1: none since reset)
  // FIBAR_TRACE=1: timing events at the stream parts' boundaries of every
  // streamed batch (fibar_debug_trace reads them; measurement only)
  bool trace = false;
  struct TraceRec {
    long long batch;
    int label;
    cudaEvent_t ev;
  };
  std::vector<TraceRec> tr;
  void mark(int label, cudaStream_t st) {
    if (!trace || tr.size() >= 200000) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, st);
    tr.push_back(TraceRec{batches, label, e});
  }
  bool temporal_on_blur = true;   // FIBAR_TEMPORAL_ON_BLUR
  int gblocks = 0;
  int long_grid_small = 48;   // FIBAR_LONG_GRID: k_temporal_long blocks for small batches
  int n_last = -1;            // the set whose anchors were enqueued last (evN)
  bool anchors_split = false;   // FIBAR_ANCHOR_STREAM=1: small batches' anchors as their own graph on nstream
  bool stage_graphs = true;   // FIBAR_STAGE_GRAPHS=0: small batches' blur stage as separate launches
  bool green_small = false;   // FIBAR_GREEN_SMALL=1: small batches' blur in the green context too
  // small batches: one CUDA graph per batch size, fed from fixed input buffers
  bool graphs_on = true;
  cudaStream_t capstream = nullptr;
  long long graph_max = 1LL << 17;
  // filter ON: small batches stream (the blur stage overlaps the next batch)
  // with their front end replayed as a graph; FIBAR_FULL_GRAPHS=1 restores
  // one whole-batch graph (serial schedule)
  bool full_graphs = false;
  std::vector<GraphEntry> graphs;
  uint16_t *gx2[NPAR] = {}, *gy2[NPAR] = {};   // fixed graph input buffers, per buffer set
  int8_t *gp2[NPAR] = {};
  int blur_grid_serial = 148;
  cudaEvent_t evF[NPAR] = {}, evB[NPAR] = {};
  cudaEvent_t evBuf[NPAR] = {};   // the set's blur stage is done (its buffers are free); evB also orders after a read-out
  int last_b = -1;   // parity of the newest batch with a blur stage in flight
  int last_par = -1;  // parity of the newest batch (fibar_debug_stale_items)
  bool b_used[NPAR] = {};
  int nsm = 148;
  int blur_grid = 148;
  int chunk = 64, warm = 64, debug = 0;
  bool warm_set = false;   // FIBAR_WARM given: used for every batch size
  int run_smem = 0;        // FIBAR_RUN_SMEM: dynamic shared memory reserved by each k_window_run block (experiment)
  bool no_reg32x = false;  // FIBAR_REG32X=0: the 64-bit regulator fix-up everywhere (measurement)
  int run_g = 8;           // FIBAR_RUN_G: lanes per chunk in the window run, small batches (0: one lane per chunk, k_window_run)
  int run_g_large = 4;     // FIBAR_RUN_G_LARGE: the same for batches above small_chunk_max
  int vf_ctas = VF_CTAS;   // FIBAR_VF_CTAS: CTAs of the verifier's cluster (<= 16)
  // batches up to this size use 32-event speculation chunks: a small batch
  // leaves most SMs idle, so shorter serial chunk runs win over the extra
  // anchors and re-runs (config 3, 100k batches: 214 -> 227 Mev/s; 1M-event
  // batches keep 64: 1173 vs 1018 Mev/s at 32).  FIBAR_CHUNK fixes one size.
  long long small_chunk_max = 1LL << 18;
  int twarm = 256;
  bool serial = false;   // FIBAR_SERIAL: blur stage on the engine stream (no overlap; for measurement)
  unsigned blur_sleep = 0;
  unsigned long long *dbg_t = nullptr, *dbg_g = nullptr;
  // halo band (filter-ON row band): rows, item lists and the batch in flight
  bool halo = false;
  int hreg0 = 0, hreg1 = 0, hin_top = -1, hin_bot = -1, hout_top = -1, hout_bot = -1;
  unsigned *hslot = nullptr, *hlist = nullptr, *hcnt = nullptr;
  int hnb = 0;
  long long hcount[4] = {0, 0, 0, 0};
  bool hopen = false;   // a halo batch awaits its rounds / finish
  Ctx hctx{};

  Ctx ctx(const unsigned *skey, const unsigned *sidx, long long n_raw, int par) const {
    Ctx x{};
    x.W = W;
    x.H = H;
    x.band_y0 = band_y0;
    x.full_H = full_H;
    x.ts = ts;
    x.tiles_x = tiles_x;
    x.A = A;
    x.n_pix = n_pix;
    x.num = cfg.fill_num;
    x.numA = cfg.fill_num * (long long)A;
    x.den = cfg.fill_den;
    x.reg32x = (x.numA < (1LL << 24) && x.den < (1LL << 24) && cfg.q_max < (1LL << 22) &&
                x.den * (cfg.q_max + 2) < (1LL << 29) && !no_reg32x) ? 1 : 0;
    x.qmin = cfg.q_min;
    x.qmax = cfg.q_max;
    x.every = cfg.regulate_every;
    x.alpha = cfg.alpha;
    x.oma = cfg.one_m_alpha;
    x.beta = cfg.beta;
    x.h = cfg.half_1p_beta;
    x.use_gain = use_gain;
    x.blur_on = blur_on;
    x.spatial = spatial;
    x.st = st;
    x.pbar = pbar;
    x.l = l;
    x.gain = gain;
    x.pt = pt2[par];
    x.plast = plast;
    x.wcnt = wcnt;
    x.bs = bsd ? bsd + par : nullptr;
    x.bsn = bsd ? bsd + (par + 1) % NPAR : nullptr;
    x.last_tile = last_tile;
    x.ptt = ptt2[par];
    x.rkey = rkey;
    x.rnext = rnext;
    x.Rm = (unsigned long long)(R - 1);
    x.raw_x = raw_x;
    x.raw_y = raw_y;
    x.raw_p = raw_p;
    x.n_raw = n_raw;
    x.n_raw_dev = nullptr;
    x.blockcnt = blockcnt2[par];
    x.ekey = ekey2[par];
    x.epol = epol2[par];
    x.spol = spol2[par];
    x.longseg = longseg2[par];
    x.max_long = (unsigned)(Bcap / LONG_SEG + 1);
    x.tkey = ka2[par];
    x.skey = skey;
    x.sidx = sidx;
    x.dp = dp2[par];
    x.S = S2[par];
    x.Qt = Qt2[par];
    x.pmap = pmap2[par];
    x.item = item2[par];
    x.posrec = posrec2[par];
    x.t2 = t2_2[par];
    x.bv64 = bv64;
    x.mv64 = mv64;
    x.prep = prep2[par];
    x.colist = colist2[par];
    x.chunk = n_raw <= small_chunk_max ? std::min(chunk, 32) : chunk;
    x.twarm = twarm;
    x.debug = debug;
    x.blur_sleep = blur_sleep;
    x.dbg_t = dbg_t;
    x.dbg_g = dbg_g;
    x.warm = (n_raw <= small_chunk_max && !warm_set) ? std::min(warm, 32) : warm;
    x.fp_fused = n_raw <= small_chunk_max ? 1 : 0;
    x.halo = halo;
    x.hreg0 = halo ? hreg0 : 0;
    x.hreg1 = halo ? hreg1 : H;
    x.hin_top = hin_top;
    x.hin_bot = hin_bot;
    x.hout_top = hout_top;
    x.hout_bot = hout_bot;
    x.hslot = hslot;
    x.hin = nullptr;
    x.anc = anc3[par];
    x.anc2 = anc23[par];
    x.anc0 = anc03[par];
    x.lc = lc3[par];
    x.lu = lu3[par];
    x.ch = ch;
    x.vl = vl;
    return x;
  }
};

namespace {

template <class T>
int dalloc(T **p, long long count) {
  if (count <= 0) count = 1;
  cudaError_t e = cudaMalloc((void **)p, sizeof(T) * (size_t)count);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  return 0;
}

// make the engine stream wait for the newest blur stage (before any read)
int join_blur(fibar_engine *g) {
  if (g->last_b >= 0) CK(cudaStreamWaitEvent(g->L.stream, g->evB[g->last_b], 0));
  return 0;
}

int init_state(fibar_engine *g) {
  cudaStream_t s = g->L.stream;
  join_blur(g);
  g->last_b = -1;
  for (bool &u : g->b_used) u = false;
  fibar_launch(g->L, "init", k_init_state, 1, 1, 0, s, g->st, g->q0, g->bsd, NPAR);
  CK(cudaMemsetAsync(g->pbar, 0, sizeof(float) * g->n_pix, s));
  CK(cudaMemsetAsync(g->l, 0, sizeof(float) * g->n_pix, s));
  if (g->spatial) {
    for (int c = 0; c < NPAR; ++c) fibar_launch(g->L, "init", k_init_pt, g->nsm * 4, TPB, 0, s, g->pt2[c], g->plast, g->n_pix);
    fibar_launch(g->L, "init", k_fill_ll, g->nsm * 4, TPB, 0, s, g->last_tile, g->n_tiles, -1);
    CK(cudaMemsetAsync(g->rkey, 0, sizeof(unsigned) * g->R, s));
    CK(cudaMemsetAsync(g->wcnt, 0, sizeof(unsigned) * g->n_pix, s));
    CK(cudaMemsetAsync(g->rnext, 0xFF, sizeof(uint2) * g->R, s));
    CK(cudaMemsetAsync(g->bv64, 0, sizeof(unsigned long long) * (g->Bcap + g->n_pix + 2), s));
    CK(cudaMemsetAsync(g->mv64, 0, sizeof(unsigned long long) * g->Bcap, s));
  }
  g->zn = 0;
  g->hfill = 0;
  g->dfill = 0;
  g->gt.n = 0;
  g->r_par = -1;
  CK(cudaGetLastError());
  return 0;
}

// The front end of a batch, in two parts.
// Ingest (stream s): the OOB filter, compaction, the pixel sort and (filter
// ON) segments and links -- it reads the batch's own events and the previous
// batch's links, never the previous window pass, so it may run ahead of it.
// Returns where the sorted pairs are.
int enqueue_ingest_a(fibar_engine *g, const uint16_t *rx0, const uint16_t *ry0, const int8_t *rp0, long long n_raw,
                     cudaEvent_t used_ev, int par, cudaStream_t s, int &where, const long long *n_dev = nullptr) {
  // part A: OOB filter, compaction, pixel sort -- the batch's own events only
  Launcher &L = g->L;
  const int nb_in = (int)((n_raw + IN_TILE - 1) / IN_TILE);
  Ctx x = g->ctx(nullptr, nullptr, n_raw, par);
  x.raw_x = rx0;
  x.raw_y = ry0;
  x.raw_p = rp0;
  x.n_raw_dev = n_dev;   // n_raw is then the size class's upper bound
  cudaStream_t s_saved = L.stream;
  L.stream = s;
  if (nb_in == 1) {
    // one tile: the block counts, scans and compacts by itself
    fibar_launch(L, "compact", k_compact, 1, TPB, 0, s, x, 1, 1);
  } else {
    fibar_launch(L, "count_inb", k_count_inb, nb_in, TPB, 0, s, x, nb_in);
    scan_exclusive_u32(L, g->blockcnt2[par], nb_in + 1);
    fibar_launch(L, "compact", k_compact, nb_in, TPB, 0, s, x, nb_in, 0);
  }
  if (used_ev) CK(cudaEventRecord(used_ev, s));   // the raw packet may be refilled / freed from here on
  where = radix_sort_pairs(L, g->ka2[par], g->va2[par], g->kb2[par], g->vb2[par], g->hist2[par], &g->bsd[par].B, n_raw,
                           g->key_bits);
  L.stream = s_saved;
  CK(cudaGetLastError());
  return 0;
}

int enqueue_ingest_b(fibar_engine *g, long long n_raw, int par, int where, cudaStream_t s) {
  // part B, in batch order: the batch's first event index, then (filter ON)
  // segments and links, which read the previous batch's links (last-touch
  // tables), never its window pass
  Launcher &L = g->L;
  cudaStream_t s_saved = L.stream;
  L.stream = s;
  Ctx x = g->ctx(where ? g->kb2[par] : g->ka2[par], where ? g->vb2[par] : g->va2[par], n_raw, par);
  if (g->spatial) {
    fibar_launch(L, "ingest_end", k_ingest_end, 1, 1, 0, s, x);
    const int nb = (int)((n_raw + TPB - 1) / TPB);
    fibar_launch(L, "seg_marks", k_seg_marks, nb, TPB, 0, s, x);
    fibar_launch(L, "link", k_link, nb, TPB, 0, s, x);
  }
  L.stream = s_saved;
  CK(cudaGetLastError());
  return 0;
}

int enqueue_ingest(fibar_engine *g, const uint16_t *rx0, const uint16_t *ry0, const int8_t *rp0, long long n_raw,
                   cudaEvent_t used_ev, int par, cudaStream_t s, int &where, const long long *n_dev = nullptr) {
  int rc = enqueue_ingest_a(g, rx0, ry0, rp0, n_raw, used_ev, par, s, where, n_dev);
  if (!rc) rc = enqueue_ingest_b(g, n_raw, par, where, s);
  return rc;
}

// The window part (stream s, after the previous batch's window part): the
// batch opens against the window state, then (filter ON) the anchors, the
// speculative run and the verifier.  Returns the batch context in x.
// The window part in two pieces.  Anchors (filter ON): exact distinct counts
// of every chunk's candidate windows, counted against the previous batch's
// predicted end state, so they may run beside the previous batch's verifier.
int enqueue_anchors(fibar_engine *g, long long n_raw, int par, int where, cudaStream_t s) {
  Launcher &L = g->L;
  Ctx x = g->ctx(where ? g->kb2[par] : g->ka2[par], where ? g->vb2[par] : g->va2[par], n_raw, par);
  // chunks 1..T: chunk T ends at the batch end (the next batch's prediction)
  const int T = (int)((n_raw + x.chunk - 1) / x.chunk);
  fibar_launch(L, "anchor", k_anchor, (int)(((long long)(T + 1) * 32 + TPB - 1) / TPB), TPB, 0, s, x);
  fibar_launch(L, "anchor_base", k_anchor_base, dim3(g->nsm / 2, NCAND), TPB, 0, s, x);
  fibar_launch(L, "anchor_scan", k_anchor_scan, NCAND + 1, 1024, 0, s, x, x.anc, NCAND);
  if (!x.fp_fused) fibar_launch(L, "fp", k_fp, (T + TPB - 1) / TPB, TPB, 0, s, x);
  fibar_launch(L, "anchor2", k_anchor2, (int)(((long long)(T + 1) * 32 + TPB - 1) / TPB), TPB, 0, s, x);
  fibar_launch(L, "anchor_scan", k_anchor_scan, NFINE, 1024, 0, s, x, x.anc2, NFINE);
  fibar_launch(L, "predict", k_predict, 1, 1, 0, s, x);
  CK(cudaGetLastError());
  return 0;
}

// ... then (after the previous batch's verifier) the speculative run and the
// verifier; ev_run (if given) is recorded between them: the next batch's
// anchors read the run's predicted end state and overwrite its candidates.
int enqueue_chain(fibar_engine *g, long long n_raw, int par, int where, cudaStream_t s, Ctx &x, cudaEvent_t ev_run) {
  Launcher &L = g->L;
  x = g->ctx(where ? g->kb2[par] : g->ka2[par], where ? g->vb2[par] : g->va2[par], n_raw, par);
  if (!g->spatial) {
    // (the batch is opened by k_compact; filter ON: by k_window_run)
  } else {
    const int T = (int)((n_raw + x.chunk - 1) / x.chunk);
    const int G = n_raw <= g->small_chunk_max ? g->run_g : g->run_g_large;
    if (G == 0) {
      fibar_launch(L, "window_run", k_window_run, (T + 127) / 128, 128, (size_t)g->run_smem, s, x);
    } else {
      // G lanes per chunk: 32 / G chunks per warp, four warps per block
      const int nbk = (int)(((long long)T * G + 127) / 128);
      if (G == 8) fibar_launch(L, "window_run", k_window_run_g8, nbk, 128, 0, s, x);
      else if (G == 4) fibar_launch(L, "window_run", k_window_run_g4, nbk, 128, 0, s, x);
      else fibar_launch(L, "window_run", k_window_run_g2, nbk, 128, 0, s, x);
    }
    // an external event-record node when captured (the next batch's anchors,
    // on another stream, wait on it)
    if (ev_run) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      CK(cudaStreamIsCapturing(s, &cs));
      if (cs == cudaStreamCaptureStatusActive)
        CK(cudaEventRecordWithFlags(ev_run, s, cudaEventRecordExternal));
      else
        CK(cudaEventRecord(ev_run, s));
    }
    // one cluster (cluster barriers between its rounds' phases)
    fibar_launch_cluster(L, "window_verify", k_window_verify, g->vf_ctas, VF_TPB, 0, s, x);
  }
  CK(cudaGetLastError());
  return 0;
}

// Both pieces on one stream.
int enqueue_window(fibar_engine *g, long long n_raw, int par, int where, cudaStream_t s, Ctx &x) {
  if (g->spatial) {
    int rc = enqueue_anchors(g, n_raw, par, where, s);
    if (rc) return rc;
  }
  return enqueue_chain(g, n_raw, par, where, s, x, nullptr);
}

// The eviction pass (stream s, after the window part; filter ON): each popped
// entry's popping event, the stale items, the per-position info; its last
// block closes the batch.  It reads only this batch's window trajectory, so it
// runs beside the next batch's window part.
int enqueue_post(fibar_engine *g, long long n_raw, int par, int where, cudaStream_t s) {
  Launcher &L = g->L;
  Ctx x = g->ctx(where ? g->kb2[par] : g->ka2[par], where ? g->vb2[par] : g->va2[par], n_raw, par);
  const int nb = (int)((n_raw + TPB - 1) / TPB);
  fibar_launch(L, "popj_map", k_popj_map, nb, TPB, 0, s, x);
  fibar_launch(L, "popj", k_popj, (int)((n_raw + TPB) / TPB) + g->nsm, TPB, 0, s, x);
  fibar_launch(L, "posinfo", k_posinfo, nb, TPB, 0, s, x, 1);   // its last block closes the batch
  CK(cudaGetLastError());
  return 0;
}

// Both parts on one stream (serial schedules, whole-batch graphs, halo bands).
int enqueue_front(fibar_engine *g, const uint16_t *rx0, const uint16_t *ry0, const int8_t *rp0, long long n_raw,
                  cudaEvent_t used_ev, int par, cudaStream_t s, Ctx &x, int &where) {
  int rc = enqueue_ingest(g, rx0, ry0, rp0, n_raw, used_ev, par, s, where);
  if (rc) return rc;
  cudaStream_t s_saved = g->L.stream;
  g->L.stream = s;
  rc = enqueue_window(g, n_raw, par, where, s, x);
  if (!rc && g->spatial) rc = enqueue_post(g, n_raw, par, where, s);
  g->L.stream = s_saved;
  x.raw_x = rx0;
  x.raw_y = ry0;
  x.raw_p = rp0;
  return rc;
}

// The temporal replay of the blur stage on stream bs: short segments there,
// long ones (listed by the ingest) beside them on tstream.
int enqueue_temporal_forked(fibar_engine *g, long long n_raw, const Ctx &x, cudaStream_t bs) {
  Launcher &L = g->L;
  const int nb = (int)((n_raw + TPB - 1) / TPB);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(bs, &cs));
  CK(cudaEventRecord(g->evT0, bs));
  CK(cudaStreamWaitEvent(g->tstream, g->evT0, 0));
  fibar_launch(L, "temporal", k_temporal_runs, nb, TPB, 0, bs, x);
  L.stream = g->tstream;
  // (a small batch has few long segments: a small grid, whose 150-register blocks need not wait for SMs)
  fibar_launch(L, "temporal_long", k_temporal_long, n_raw <= g->small_chunk_max ? g->long_grid_small : g->nsm * 2, LONG_TPB, 0,
               g->tstream, x);
  CK(cudaEventRecord(g->evT1, g->tstream));
  CK(cudaStreamWaitEvent(bs, g->evT1, 0));
  L.stream = bs;
  return 0;
}

// The rest of the blur stage (no green context: small batches)
int enqueue_blur_rest(fibar_engine *g, long long n_raw, const Ctx &x, cudaStream_t bs, bool graph) {
  Launcher &L = g->L;
  L.stream = bs;
  if (g->blur_on) {
    const int nbp = (int)((n_raw + TPB) / TPB) + g->nsm;
    fibar_launch(L, "blur_prep", k_blur_prep, nbp, TPB, 0, bs, x);
    fibar_launch(L, "blur", k_blur, graph ? g->blur_grid_serial : g->blur_grid, TPB, 0, bs, x);
  }
  fibar_launch(L, "final", k_final, g->nsm * 8, TPB, 0, bs, x);
  return 0;
}

// the blur stage of a small batch as captured into its graph (stream: capstream)
int capture_blur_stage(fibar_engine *g, long long n_raw, int par, int where) {
  Ctx x = g->ctx(where ? g->kb2[par] : g->ka2[par], where ? g->vb2[par] : g->va2[par], n_raw, par);
  x.raw_x = g->gx2[par];
  x.raw_y = g->gy2[par];
  x.raw_p = g->gp2[par];
  int rc = enqueue_temporal_forked(g, n_raw, x, g->capstream);
  if (!rc) rc = enqueue_blur_rest(g, n_raw, x, g->capstream, false);
  return rc;
}

// The captured front end for a size class (n_raw: the class's upper bound)
// and a parity, as two graphs: exec the ingest (reading the fixed input
// buffers gx/gy/gp and the batch's raw count that k_stage leaves in the
// batch state), exec2 the window part.  Every kernel reads the batch's real
// counts from device memory, so one capture serves the whole class.  One
// cache entry holds both graphs, so evicting an entry never splits a pair.
// Captured on first use (nullptr on failure).
GraphEntry *front_graph(fibar_engine *g, long long n_raw, int par) {
  for (auto &ge : g->graphs)
    if (ge.kind == 1 && ge.n == n_raw && ge.par == par) return &ge;
  if (g->graphs.size() >= 8 * NPAR) {   // small cache: drop the oldest (freed once its launches finish)
    for (cudaGraphExec_t e : {g->graphs.front().exec, g->graphs.front().exec2, g->graphs.front().exec3,
                              g->graphs.front().exec4, g->graphs.front().exec5, g->graphs.front().exec6})
      if (e) cudaGraphExecDestroy(e);
    g->graphs.erase(g->graphs.begin());
  }
  if (!g->capstream && cudaStreamCreateWithFlags(&g->capstream, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  Launcher &L = g->L;
  cudaStream_t s0 = L.stream;
  GraphEntry ge;
  ge.n = n_raw;
  ge.kind = 1;
  ge.par = par;
  for (int part : {0, 1, 2, 3, 4, 5}) {
    if (part == 3 && !g->anchors_split) continue;   // (the anchors ride in the links' graph)
    const long long l0 = L.launches;
    cudaGraph_t graph = nullptr;
    Ctx x{};
    const auto t_c0 = std::chrono::steady_clock::now();
    if (cudaStreamBeginCapture(g->capstream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      for (cudaGraphExec_t e : {ge.exec, ge.exec2, ge.exec3, ge.exec4, ge.exec5, ge.exec6})
        if (e) cudaGraphExecDestroy(e);
      return nullptr;
    }
    L.stream = g->capstream;
    const int rc = part == 0   ? enqueue_ingest_a(g, g->gx2[par], g->gy2[par], g->gp2[par], n_raw, nullptr, par,
                                                  g->capstream, ge.where, &g->bsd[par].n_raw)
                   : part == 4 ? (enqueue_ingest_b(g, n_raw, par, ge.where, g->capstream) ||
                                  (g->anchors_split ? 0 : enqueue_anchors(g, n_raw, par, ge.where, g->capstream)))
                   : part == 5 ? capture_blur_stage(g, n_raw, par, ge.where)
                   : part == 1 ? enqueue_chain(g, n_raw, par, ge.where, g->capstream, x, nullptr)
                   : part == 2 ? enqueue_post(g, n_raw, par, ge.where, g->capstream)
                               : enqueue_anchors(g, n_raw, par, ge.where, g->capstream);
    L.stream = s0;
    const auto t_c1 = std::chrono::steady_clock::now();
    cudaError_t ce = cudaStreamEndCapture(g->capstream, &graph);
    cudaGraphExec_t exec = nullptr;
    if (rc == 0 && ce == cudaSuccess) ce = cudaGraphInstantiate(&exec, graph, 0);
    if (getenv("FIBAR_DEBUG_CAPTURE")) {
      const auto t_c2 = std::chrono::steady_clock::now();
      fprintf(stderr, "[fibar] capture part %d par %d n %lld: capture %.3f ms, end+instantiate %.3f ms\n", part, par, n_raw,
              std::chrono::duration<double, std::milli>(t_c1 - t_c0).count(),
              std::chrono::duration<double, std::milli>(t_c2 - t_c1).count());
    }
    if (graph) cudaGraphDestroy(graph);
    const long long k = L.launches - l0;
    L.launches = l0;
    if (rc || ce != cudaSuccess) {
      cudaGetLastError();
      for (cudaGraphExec_t e : {ge.exec, ge.exec2, ge.exec3, ge.exec4, ge.exec5, ge.exec6})
        if (e) cudaGraphExecDestroy(e);
      g->graphs_on = false;   // capture impossible here: stream every kernel from now on
      return nullptr;
    }
    if (part == 0) {
      ge.exec = exec;
      ge.kernels = k;
    } else if (part == 1) {
      ge.exec2 = exec;
      ge.kernels2 = k;
    } else if (part == 2) {
      ge.exec3 = exec;
      ge.kernels3 = k;
    } else if (part == 3) {
      ge.exec4 = exec;
      ge.kernels4 = k;
    } else if (part == 4) {
      ge.exec5 = exec;
      ge.kernels5 = k;
    } else {
      ge.exec6 = exec;
      ge.kernels6 = k;
    }
  }
  g->graphs.push_back(ge);
  return &g->graphs.back();
}

// Enqueue one device batch.  graph == false: the streamed form (blur stage on
// the second stream, cross-batch events).  graph == true: everything on the
// engine stream with parity-0 buffers and no events, the form captured into a
// CUDA graph for small batches (see run_batch_raw).
//
// Streamed, filter ON: the front end's two parts run on the engine's own
// streams.  The ingest (astream) waits for the packet (the caller's stream at
// the call) and for its parity's buffers (the blur stage two batches back);
// the window part (fstream) waits for the ingest and runs after the previous
// batch's window part.  So batch k+1's ingest and sort overlap batch k's
// window pass.  The caller's stream waits for the ingest's read of the packet.
int enqueue_batch(fibar_engine *g, const uint16_t *rx0, const uint16_t *ry0, const int8_t *rp0, long long n_raw,
                  cudaEvent_t used_ev, int par, bool graph) {
  Launcher &L = g->L;
  const cudaStream_t u = L.stream;   // the caller's stream
  g->last_par = par;
  const bool split = !graph && g->spatial && !g->serial && !g->halo && g->temporal_on_blur;
  cudaStream_t s = split ? g->fstream : u;   // the window part's stream
  Ctx x{};
  int where = 0;
  const int nb = (int)((n_raw + TPB - 1) / TPB);
  const GraphEntry *stage_graph = nullptr;   // small batches: the blur stage's graph
  if (split) {
    const bool small = g->graphs_on && !L.prof && n_raw <= g->graph_max;
    // a small batch's sort part alternates between two streams
    const int lane_i = small ? (int)(g->batches % g->sort_lanes) : 0;
    cudaStream_t sa = lane_i == 0 ? g->astream : (lane_i == 1 ? g->astream2 : g->astream3);
    CK(cudaEventRecord(g->evIn, u));
    CK(cudaStreamWaitEvent(sa, g->evIn, 0));
    if (g->b_used[par]) CK(cudaStreamWaitEvent(sa, g->evBuf[par], 0));   // this parity's buffers are free (the ingest reads no brightness: it need not wait for a read-out)
    g->mark(0, sa);   // trace labels: 0/1 ingest start/end, 2/3 window part, 4/5 eviction pass, 6/7 blur stage
    if (small) {
      // a small batch: each part replays one CUDA graph per (size class,
      // parity), the ingest from fixed input buffers (k_stage fills them and
      // the batch's raw count)
      // (a class of its own for packets of up to one sort tile: sorted on chip by one CTA)
      const long long cls = n_raw <= 2048 ? std::min(g->graph_max, 2048LL)
                                          : std::min(g->graph_max, (n_raw + GRAPH_CLASS - 1) / GRAPH_CLASS * GRAPH_CLASS);
      const int nbs = (int)std::max(1LL, std::min((long long)g->nsm * 2, (n_raw / 8 + TPB - 1) / TPB));
      fibar_launch(L, "stage", k_stage, nbs, TPB, 0, sa, rx0, ry0, rp0, (long long)n_raw, g->gx2[par], g->gy2[par],
                   g->gp2[par], &g->bsd[par].n_raw);
      CK(cudaEventRecord(g->evCp, sa));
      if (used_ev) CK(cudaEventRecord(used_ev, sa));
      const GraphEntry *ge = front_graph(g, cls, par);
      if (!ge) return g_err.empty() ? fail(FIBAR_E_CUDA, "front-end graph capture failed") : FIBAR_E_CUDA;
      where = ge->where;
      CK(cudaGraphLaunch(ge->exec, sa));
      L.launches += ge->kernels;
      CK(cudaEventRecord(g->evS[par], sa));
      // segments and links in batch order
      CK(cudaStreamWaitEvent(g->lstream, g->evS[par], 0));
      // the anchors read the start state the previous batch's anchors predicted
      // (a large batch's run on nstream)
      if (!g->anchors_split && g->n_last >= 0) CK(cudaStreamWaitEvent(g->lstream, g->evN[g->n_last], 0));
      CK(cudaGraphLaunch(ge->exec5, g->lstream));
      L.launches += ge->kernels5;
      g->mark(1, g->lstream);
      if (g->anchors_split) {
        // the anchors on their own stream: the links of the next batch need not wait for them
        CK(cudaEventRecord(g->evA[par], g->lstream));
        CK(cudaStreamWaitEvent(g->nstream, g->evA[par], 0));
        if (g->n_last >= 0) CK(cudaStreamWaitEvent(g->nstream, g->evN[g->n_last], 0));
        CK(cudaGraphLaunch(ge->exec4, g->nstream));
        L.launches += ge->kernels4;
        CK(cudaEventRecord(g->evN[par], g->nstream));
      } else {
        // (the same graph carries the anchors: they follow the previous batch's anyway)
        CK(cudaEventRecord(g->evN[par], g->lstream));
      }
      g->n_last = par;
      CK(cudaStreamWaitEvent(s, g->evN[par], 0));
      if (g->stage_graphs && !g->green_small) stage_graph = ge;
      g->mark(2, s);
      CK(cudaGraphLaunch(ge->exec2, s));   // (records evR[par] after the run)
      L.launches += ge->kernels2;
      g->r_par = par;
      g->mark(3, s);
      CK(cudaEventRecord(g->evV[par], s));
      CK(cudaStreamWaitEvent(g->pstream, g->evV[par], 0));
      g->mark(4, g->pstream);
      CK(cudaGraphLaunch(ge->exec3, g->pstream));
      L.launches += ge->kernels3;
      g->mark(5, g->pstream);
      x = g->ctx(where ? g->kb2[par] : g->ka2[par], where ? g->vb2[par] : g->va2[par], n_raw, par);
      x.raw_x = g->gx2[par];
      x.raw_y = g->gy2[par];
      x.raw_p = g->gp2[par];
    } else {
      int rc = enqueue_ingest_a(g, rx0, ry0, rp0, n_raw, used_ev, par, sa, where);
      if (rc) return rc;
      CK(cudaEventRecord(g->evCp, sa));
      // segments and links on lstream, where every batch's run in batch order
      CK(cudaEventRecord(g->evS[par], sa));
      CK(cudaStreamWaitEvent(g->lstream, g->evS[par], 0));
      rc = enqueue_ingest_b(g, n_raw, par, where, g->lstream);
      if (rc) return rc;
      g->mark(1, g->lstream);
      CK(cudaEventRecord(g->evA[par], g->lstream));
      cudaStream_t sn = g->nstream;
      CK(cudaStreamWaitEvent(sn, g->evA[par], 0));
      if (g->n_last >= 0) CK(cudaStreamWaitEvent(sn, g->evN[g->n_last], 0));   // (a small batch's anchors ran on lstream)
      L.stream = sn;
      rc = enqueue_anchors(g, n_raw, par, where, sn);
      L.stream = u;
      if (rc) return rc;
      CK(cudaEventRecord(g->evN[par], sn));
      g->n_last = par;
      CK(cudaStreamWaitEvent(s, g->evN[par], 0));
      L.stream = s;
      rc = enqueue_chain(g, n_raw, par, where, s, x, nullptr);
      L.stream = u;
      if (rc) return rc;
      g->r_par = par;
      CK(cudaEventRecord(g->evV[par], s));
      CK(cudaStreamWaitEvent(g->pstream, g->evV[par], 0));
      L.stream = g->pstream;
      rc = enqueue_post(g, n_raw, par, where, g->pstream);
      L.stream = u;
      if (rc) return rc;
      x.raw_x = rx0;
      x.raw_y = ry0;
      x.raw_p = rp0;
    }
    CK(cudaStreamWaitEvent(u, g->evCp, 0));   // the caller may reuse the packet after the ingest read it
    s = g->pstream;   // the batch's front end ends with the eviction pass
    L.stream = s;
  } else {
    // this parity's buffers are free once the batch two back finished its blur stage
    if (!graph && g->spatial && g->b_used[par]) CK(cudaStreamWaitEvent(s, g->evB[par], 0));
    int rc = enqueue_front(g, rx0, ry0, rp0, n_raw, used_ev, par, s, x, where);
    if (rc) return rc;
  }
  if (g->spatial) {
    // The batch's counters (event count, stale count, candidate set) closed
    // at the end of the window part (k_posinfo): the next front end reads
    // them.  Its links read the last-touch tables, which k_link already
    // advanced; so the next front end never waits for this batch's temporal
    // replay or blur stage (only, two batches on, for its parity's buffers).
    // The temporal replay reads the brightness the previous batch's blur
    // stage finishes.  Streamed (temporal_on_blur): it runs first on the blur
    // stream itself, so the cycle blur(k) -> final(k) -> replay(k+1) ->
    // prep(k+1) -> blur(k+1) crosses no stream.
    const bool t_on_b = !graph && !g->serial && !g->halo && g->temporal_on_blur;
    if (t_on_b) {
      cudaStream_t bs = g->bstream;
      CK(cudaEventRecord(g->evF[par], s));
      CK(cudaStreamWaitEvent(bs, g->evF[par], 0));
      g->mark(6, bs);
      if (stage_graph) {
        // a small batch: the whole blur stage replays one graph
        CK(cudaGraphLaunch(stage_graph->exec6, bs));
        L.launches += stage_graph->kernels6;
        L.stream = u;
        g->mark(7, bs);
        CK(cudaEventRecord(g->evB[par], bs));
        CK(cudaEventRecord(g->evBuf[par], bs));
        g->b_used[par] = true;
        g->last_b = par;
        CK(cudaGetLastError());
        return 0;
      }
      L.stream = bs;
      int rc = enqueue_temporal_forked(g, n_raw, x, bs);
      if (rc) return rc;
    } else {
      if (!graph && g->last_b >= 0) CK(cudaStreamWaitEvent(s, g->evB[g->last_b], 0));
      fibar_launch(L, "temporal", k_temporal_runs, nb, TPB, 0, s, x);
      fibar_launch(L, "temporal_long", k_temporal_long, g->nsm * 2, LONG_TPB, 0, s, x);
    }
    if (g->halo) {
      // halo band: the item lists of the exchanged rows and the tap
      // resolution; the host then drives the blur rounds (fibar_halo_round)
      const int nbh = (int)((n_raw + g->n_pix + 2 + TPB - 1) / TPB);
      fibar_launch(L, "halo_count", k_halo_count, nbh, TPB, 0, s, x, g->hcnt, nbh);
      scan_exclusive_u32(L, g->hcnt, 4 * nbh + 1);
      fibar_launch(L, "halo_write", k_halo_write, nbh, TPB, 0, s, x, (const unsigned *)g->hcnt, nbh, g->hlist);
      const int nbp = (int)((n_raw + TPB) / TPB) + g->nsm;
      fibar_launch(L, "blur_prep", k_blur_prep, nbp, TPB, 0, s, x);
      g->hnb = nbh;
      g->hctx = x;
      L.stream = u;
      CK(cudaGetLastError());
      return 0;
    }
    // blur stage on its own stream: overlaps the next batch's front end
    cudaStream_t bs = (g->serial || graph) ? s : g->bstream;
    if (!graph && !t_on_b) {
      CK(cudaEventRecord(g->evF[par], s));
      CK(cudaStreamWaitEvent(bs, g->evF[par], 0));
    }
    L.stream = bs;
    if (g->blur_on) {
      const int nbp = (int)((n_raw + TPB) / TPB) + g->nsm;
      fibar_launch(L, "blur_prep", k_blur_prep, nbp, TPB, 0, bs, x);
      if (g->gstream && !graph && (n_raw > g->small_chunk_max || g->green_small)) {
        // the blur dataflow alone on its own SM partition (green context):
        // its polling no longer shares SMs with the next batch's front end
        // (large batches; a small batch's blur stage is the critical chain
        // and takes the whole GPU: config 3, 374 -> 389 Mev/s)
        CK(cudaEventRecord(g->evP, bs));
        CK(cudaStreamWaitEvent(g->gstream, g->evP, 0));
        L.stream = g->gstream;
        fibar_launch(L, "blur", k_blur, g->gblocks, TPB, 0, g->gstream, x);
        CK(cudaEventRecord(g->evG, g->gstream));
        CK(cudaStreamWaitEvent(bs, g->evG, 0));
        L.stream = bs;
      } else {
        fibar_launch(L, "blur", k_blur, graph ? g->blur_grid_serial : g->blur_grid, TPB, 0, bs, x);
      }
    }
    fibar_launch(L, "final", k_final, g->nsm * 8, TPB, 0, bs, x);
    L.stream = u;
    if (!graph) {
      g->mark(7, bs);
      CK(cudaEventRecord(g->evB[par], bs));
      CK(cudaEventRecord(g->evBuf[par], bs));
      g->b_used[par] = true;
      g->last_b = par;
    }
  } else {
    fibar_launch(L, "posinfo", k_posinfo, nb, TPB, 0, s, x, 0);
    fibar_launch(L, "temporal", k_temporal, nb, TPB, 0, s, x);
    fibar_launch(L, "temporal_long", k_temporal_long, g->nsm * 2, LONG_TPB, 0, s, x);
    // (the event count was added by k_compact)
  }
  L.stream = u;
  CK(cudaGetLastError());
  return 0;
}

// A small batch is launch-bound (~45 dependent kernels doing a few us of work
// each), so it runs as one CUDA graph per batch size: its inputs are copied
// into fixed graph buffers, the kernel sequence is captured once per size and
// replayed with a single launch.  Large batches stream (two-stream overlap).
int run_batch_raw(fibar_engine *g, const uint16_t *rx0, const uint16_t *ry0, const int8_t *rp0, long long n_raw,
                  cudaEvent_t used_ev) {
  if (n_raw <= 0) return 0;
  Launcher &L = g->L;
  cudaStream_t s = L.stream;
  if (!g->graphs_on || L.prof || n_raw > g->graph_max || !g->full_graphs) {
    const int par = g->spatial ? (int)(g->batches % NPAR) : 0;
    int rc = enqueue_batch(g, rx0, ry0, rp0, n_raw, used_ev, par, false);
    if (rc) return rc;
    g->batches++;
    return 0;
  }
  // graph form: after every earlier blur stage (it reuses parity-0 buffers)
  join_blur(g);
  g->last_b = -1;
  for (bool &u : g->b_used) u = false;
  CK(cudaMemcpyAsync(g->gx2[0], rx0, sizeof(uint16_t) * n_raw, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(g->gy2[0], ry0, sizeof(uint16_t) * n_raw, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(g->gp2[0], rp0, sizeof(int8_t) * n_raw, cudaMemcpyDeviceToDevice, s));
  if (used_ev) CK(cudaEventRecord(used_ev, s));   // the raw staging may be refilled from here on
  GraphEntry *hit = nullptr;
  for (auto &ge : g->graphs)
    if (ge.kind == 0 && ge.n == n_raw) hit = &ge;
  if (!hit) {
    if (g->graphs.size() >= 8) {   // small cache: drop the oldest size
      cudaGraphExecDestroy(g->graphs.front().exec);
      if (g->graphs.front().exec2) cudaGraphExecDestroy(g->graphs.front().exec2);
      g->graphs.erase(g->graphs.begin());
    }
    // captured on a private stream (the caller's may be the legacy default
    // stream, which cannot be captured); replayed on the caller's
    cudaGraph_t graph = nullptr;
    const long long l0 = L.launches;
    if (!g->capstream) CK(cudaStreamCreateWithFlags(&g->capstream, cudaStreamNonBlocking));
    cudaError_t ce = cudaStreamBeginCapture(g->capstream, cudaStreamCaptureModeThreadLocal);
    int rc = 0;
    if (ce == cudaSuccess) {
      L.stream = g->capstream;
      rc = enqueue_batch(g, g->gx2[0], g->gy2[0], g->gp2[0], n_raw, nullptr, 0, true);
      L.stream = s;
      ce = cudaStreamEndCapture(g->capstream, &graph);
    }
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    GraphEntry ge;
    ge.n = n_raw;
    ge.kernels = L.launches - l0;
    L.launches = l0;
    if (ce == cudaSuccess) {
      ce = cudaGraphInstantiate(&ge.exec, graph, 0);
      cudaGraphDestroy(graph);
    }
    if (ce != cudaSuccess) {
      // capture not possible here (e.g. the calling thread is itself capturing
      // in global mode): run the same serial schedule without a graph from now on
      cudaGetLastError();
      g->graphs_on = false;
      rc = enqueue_batch(g, g->gx2[0], g->gy2[0], g->gp2[0], n_raw, nullptr, 0, true);
      if (rc) return rc;
      g->batches++;
      return 0;
    }
    g->graphs.push_back(ge);
    hit = &g->graphs.back();
  }
  CK(cudaGraphLaunch(hit->exec, s));
  L.launches += hit->kernels;
  g->last_par = 0;   // whole-batch graphs use the parity-0 buffers
  g->batches++;
  return 0;
}

// hand the filled host staging set to the device and run it
// pinned host packets of at least half a device batch skip the CPU staging
// copy (smaller ones are coalesced through the staging buffers as before)
long long direct_min(const fibar_engine *g) { return std::max(1LL << 16, g->Bcap / 2); }

bool is_pinned(const void *ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int launch_host_batch(fibar_engine *g) {
  if (g->hfill == 0) return 0;
  const int c = g->cur;
  const long long n = g->hfill;
  CK(cudaStreamWaitEvent(g->cstream, g->ev_used[c], 0));
  CK(cudaMemcpyAsync(g->sx[c], g->hx[c], sizeof(uint16_t) * n, cudaMemcpyHostToDevice, g->cstream));
  CK(cudaMemcpyAsync(g->sy[c], g->hy[c], sizeof(uint16_t) * n, cudaMemcpyHostToDevice, g->cstream));
  CK(cudaMemcpyAsync(g->sp_[c], g->hp[c], sizeof(int8_t) * n, cudaMemcpyHostToDevice, g->cstream));
  CK(cudaEventRecord(g->ev_h2d[c], g->cstream));
  CK(cudaStreamWaitEvent(g->L.stream, g->ev_h2d[c], 0));
  g->hfill = 0;
  g->cur ^= 1;
  return run_batch_raw(g, g->sx[c], g->sy[c], g->sp_[c], n, g->ev_used[c]);
}

// gather the pending device packets into staging set `cur` and run them
int flush_gather(fibar_engine *g) {
  if (g->dfill == 0) return 0;
  const int c = g->cur;
  const long long n = g->dfill;
  Launcher &L = g->L;
  CK(cudaStreamWaitEvent(L.stream, g->ev_used[c], 0));   // the staging set's previous batch has read it
  // enough CTAs per packet for ~16k events each, up to the SM count
  long long biggest = 0;
  for (int i = 0; i < g->gt.n; ++i) biggest = std::max(biggest, g->gt.e[i].n);
  const int per = (int)std::max(1LL, std::min((long long)g->nsm, (biggest + 16383) / 16384));
  fibar_launch(L, "gather", k_gather, dim3(per, g->gt.n), TPB, 0, L.stream, g->gt, g->sx[c], g->sy[c], g->sp_[c]);
  g->gt.n = 0;
  g->dfill = 0;
  g->cur ^= 1;
  return run_batch_raw(g, g->sx[c], g->sy[c], g->sp_[c], n, g->ev_used[c]);
}

// add a device packet (part) to the gather table
int gather_add(fibar_engine *g, const uint16_t *x, const uint16_t *y, const int8_t *p, long long n) {
  GatherTable &t = g->gt;
  if (t.n > 0) {   // contiguous with the previous entry: extend it
    GatherEntry &e = t.e[t.n - 1];
    if (x == e.x + e.n && y == e.y + e.n && p == e.p + e.n) {
      e.n += n;
      g->dfill += n;
      return 0;
    }
  }
  t.e[t.n++] = GatherEntry{x, y, p, n, g->dfill};
  g->dfill += n;
  return 0;
}

// run everything pending (zero-copy device range or gathered device packets,
// then staged host packets)
int run_batch(fibar_engine *g) {
  if (g->dfill > 0) {
    int rc = flush_gather(g);
    if (rc) return rc;
  }
  if (g->zn > 0) {
    const long long n = g->zn;
    g->zn = 0;
    int rc = run_batch_raw(g, g->zx, g->zy, g->zp, n, nullptr);
    if (rc) return rc;
  }
  return launch_host_batch(g);
}

// run everything pending and order the engine stream after the blur stage
int sync_point(fibar_engine *g) {
  int rc = run_batch(g);
  if (rc) return rc;
  return join_blur(g);
}

// read-out (pipeline.py:247-269) of n float32 values at l: exact order
// statistics for the robust bounds (numpy 'linear' percentile), float64 map
int render_core(Launcher &L, const float *l, long long n, int32_t mode, double fixed_bound, uint8_t *out,
                int32_t out_mem, double *bounds, int32_t *degenerate, SelState *sel, uint8_t *frame, int nsm) {
  if (mode == FIBAR_RENDER_FIXED && !(fixed_bound > 0)) return fail(FIBAR_E_CONFIG, "fixed scale bound must be positive");
  if (mode != FIBAR_RENDER_FIXED && mode != FIBAR_RENDER_ROBUST) return fail(FIBAR_E_CONFIG, "unknown scale mode");
  cudaStream_t s = L.stream;
  double g_lo = 0, g_hi = 0;
  uint4 ranks = make_uint4(0u, 0u, 0u, 0u);
  if (mode == FIBAR_RENDER_ROBUST) {
    // virtual index (n-1)*q, neighbours floor / floor+1, clamped at the top
    const double qs[2] = {1.0 / 100.0, 99.0 / 100.0};
    double gam[2];
    unsigned rk[4];
    for (int t = 0; t < 2; ++t) {
      const double v = (double)(n - 1) * qs[t];
      long long prev, next;
      if (v >= (double)(n - 1)) {
        prev = next = n - 1;
        gam[t] = v + 1.0;   // numpy's gamma uses index -1 here; a == b so the value is unaffected
      } else if (v < 0) {
        prev = next = 0;
        gam[t] = v;
      } else {
        prev = (long long)std::floor(v);
        next = prev + 1;
        gam[t] = v - (double)prev;
      }
      rk[2 * t] = (unsigned)prev;
      rk[2 * t + 1] = (unsigned)next;
    }
    g_lo = gam[0];
    g_hi = gam[1];
    ranks = make_uint4(rk[0], rk[1], rk[2], rk[3]);
  }
  uint8_t *dst = out_mem == FIBAR_MEM_DEVICE ? out : frame;
  // one cooperative launch, one CTA per SM (fewer for small grids), each CTA
  // holding its slice of keys on chip when it fits (k_readout)
  const long long grid0 = std::max(1LL, std::min((long long)nsm, (n + 2047) / 2048));
  const long long slice = ((n + grid0 - 1) / grid0 + 3) & ~3LL;
  const int grid = (int)((n + slice - 1) / slice);
  const int on_chip = slice * 4 <= RO_SMEM_MAX ? 1 : 0;
  {
    static unsigned long long attr_set = 0;   // per device: dynamic shared memory opt-in done
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !(attr_set >> dev & 1ull)) {
      CK(cudaFuncSetAttribute(k_readout, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RO_SMEM_MAX));
      attr_set |= 1ull << dev;
    }
  }
  L.begin("readout");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(RO_TPB);
  cfg.dynamicSmemBytes = on_chip ? (size_t)slice * 4 : 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_readout, l, (long long)n, sel, (int)mode, fixed_bound, ranks, g_lo, g_hi, dst, slice,
                        on_chip));
  L.end();
  CK(cudaGetLastError());
  if (out_mem != FIBAR_MEM_DEVICE) CK(cudaMemcpyAsync(out, frame, n, cudaMemcpyDeviceToHost, s));
  if (bounds || degenerate || out_mem != FIBAR_MEM_DEVICE) {
    struct {
      double lo, hi;
      int degenerate;
    } h;
    CK(cudaMemcpyAsync(&h, &sel->lo, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (bounds) {
      bounds[0] = h.lo;
      bounds[1] = h.hi;
    }
    if (degenerate) *degenerate = h.degenerate;
  }
  return 0;
}

}  // namespace

// ------------------------------------------------------------------ C ABI ---

extern "C" {

const char *fibar_last_error(void) { return g_err.c_str(); }

int fibar_create(const fibar_config *cfg, void *stream, fibar_engine **out) {
  if (!cfg || !out) return fail(FIBAR_E_CONFIG, "null argument");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(FIBAR_E_NODEVICE, "no CUDA device");
  // the window verifier is one 16-CTA cluster (beyond the portable 8)
  CK(cudaFuncSetAttribute(k_window_verify, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));

  if (cfg->width < 2 || cfg->height < 2) return fail(FIBAR_E_CONFIG, "geometry must be at least 2x2");
  if (cfg->tile_side < 2) return fail(FIBAR_E_CONFIG, "tile_side must be >= 2");
  if (cfg->regulate_every < 1) return fail(FIBAR_E_CONFIG, "regulate_every must be >= 1");
  const long long n = (long long)cfg->width * cfg->height;
  if (cfg->q_max > n) return fail(FIBAR_E_CONFIG, "q_max exceeds pixel count");
  if (cfg->q_min < 1 || cfg->q_min > cfg->q_max) return fail(FIBAR_E_CONFIG, "bad q_min/q_max");
  if (cfg->fill_num < 1 || cfg->fill_den < 1) return fail(FIBAR_E_CONFIG, "bad fill ratio");
  if (cfg->width > 65535 || cfg->height > 65535) return fail(FIBAR_E_CONFIG, "coordinates must fit uint16");
  if (cfg->sensor_height > 0) {
    if (cfg->band_y0 < 0 || cfg->band_y0 + cfg->height > cfg->sensor_height)
      return fail(FIBAR_E_CONFIG, "row band outside the sensor");
    if (cfg->spatial_enabled && (cfg->band_y0 != 0 || cfg->height != cfg->sensor_height))
      return fail(FIBAR_E_CONFIG, "row bands need the spatial filter off (the window is one global FIFO)");
  }
  const bool halo = cfg->halo_own_y1 > 0;
  if (halo) {
    const int y0 = cfg->halo_own_y0, y1 = cfg->halo_own_y1, G = cfg->halo_rows, Hh = cfg->height;
    if (!cfg->spatial_enabled || !cfg->blur_enabled)
      return fail(FIBAR_E_CONFIG, "halo bands are for the spatial filter with blur (filter OFF: row bands)");
    if (cfg->sensor_height > 0) return fail(FIBAR_E_CONFIG, "halo band and filter-OFF row band are exclusive");
    if (y0 < 0 || y1 > Hh || y0 >= y1) return fail(FIBAR_E_CONFIG, "halo band rows outside the sensor");
    if (G < 1 || G > y1 - y0) return fail(FIBAR_E_CONFIG, "halo rows must be in [1, band rows]");
    if ((y0 > 0 && y0 - G < 0) || (y1 < Hh && y1 + G > Hh))
      return fail(FIBAR_E_CONFIG, "halo rows exceed the neighbouring band");
  }
  fibar_engine *g = new fibar_engine();
  g->cfg = *cfg;
  if (halo) {
    const int y0 = cfg->halo_own_y0, y1 = cfg->halo_own_y1, G = cfg->halo_rows, Hh = cfg->height;
    g->halo = true;
    g->hreg0 = std::max(0, y0 - G);
    g->hreg1 = std::min(Hh, y1 + G);
    g->hin_top = y0 > 0 ? y0 - G : -1;
    g->hin_bot = y1 < Hh ? y1 + G - 1 : -1;
    g->hout_top = y0 > 0 ? y0 + G - 1 : -1;
    g->hout_bot = y1 < Hh ? y1 - G : -1;
    g->serial = true;        // every kernel on the engine stream (rounds are host driven)
    g->graphs_on = false;
  }
  g->cfg.gain = nullptr;
  g->W = cfg->width;
  g->H = cfg->height;
  g->band_y0 = (unsigned)cfg->band_y0;
  g->full_H = cfg->sensor_height > 0 ? (unsigned)cfg->sensor_height : (unsigned)cfg->height;
  g->ts = cfg->tile_side;
  g->A = g->ts * g->ts;
  g->tiles_x = (g->W + g->ts - 1) / g->ts;
  g->tiles_y = (g->H + g->ts - 1) / g->ts;
  g->n_pix = n;
  g->n_tiles = (long long)g->tiles_x * g->tiles_y;
  g->q0 = std::min(std::max(n / 16, (long long)cfg->q_min), (long long)cfg->q_max);
  g->L.stream = (cudaStream_t)stream;
  g->spatial = cfg->spatial_enabled != 0;
  g->blur_on = cfg->blur_enabled != 0;
  g->use_gain = cfg->gain != nullptr;
  // (round 1, 4 events per pixel, Mev/s: 1280x720 with one read-out 816 / 945 / 986 at 1M / 2M /
  // 3.7M; 640x480 1122 / 1213 / 1210 / 1197 at 768k / 1M / 1.2M / 1.5M -- the front end paced a batch then)
  // default device batch: 2 events per pixel (the blur stage paces large batches, and its DAG
  // deepens with the batch: 640x480 1178 -> 1222 Mev/s, 1280x720 1222 -> 1283 against 4 per pixel)
  // (filter OFF has no blur DAG: 4 per pixel, at least 1M)
  const long long bauto = cfg->spatial_enabled ? std::min(6LL << 20, std::max(1LL << 19, (2 * n + 65535) / 65536 * 65536))
                                              : std::min(6LL << 20, std::max(1LL << 20, (4 * n + 65535) / 65536 * 65536));
  g->Bcap = cfg->batch_capacity > 0 ? cfg->batch_capacity : bauto;
  if (g->Bcap > (1LL << 28)) g->Bcap = 1LL << 28;
  if (g->Bcap < 1024) g->Bcap = std::max(g->Bcap, 16LL);
  g->key_bits = ceil_log2(g->n_tiles * g->A);
  // window-speculation tuning knobs (results never depend on them; the verifier
  // re-runs any chunk whose speculative start was wrong)
  if (const char *v = getenv("FIBAR_CHUNK")) {
    g->chunk = std::max(CHUNK_MIN, atoi(v));
    g->small_chunk_max = 0;
  }
  // small batches (<= small_chunk_max) warm up 32 events: the verifier
  // re-runs the extra misses cheaply (config 3: 270 -> 280 Mev/s)
  if (const char *v = getenv("FIBAR_TRACE")) g->trace = atoi(v) != 0;
  if (const char *v = getenv("FIBAR_REG32X")) g->no_reg32x = atoi(v) == 0;
  if (const char *v = getenv("FIBAR_RUN_G")) g->run_g = atoi(v);
  if (const char *v = getenv("FIBAR_RUN_G_LARGE")) g->run_g_large = atoi(v);
  for (int *gg : {&g->run_g, &g->run_g_large}) *gg = *gg >= 8 ? 8 : (*gg >= 4 ? 4 : (*gg >= 2 ? 2 : 0));
  if (const char *v = getenv("FIBAR_VF_CTAS")) g->vf_ctas = std::min(16, std::max(1, atoi(v)));
  if (const char *v = getenv("FIBAR_RUN_SMEM")) {
    g->run_smem = std::max(0, atoi(v));
    if (g->run_smem > 48 * 1024) cudaFuncSetAttribute(k_window_run, cudaFuncAttributeMaxDynamicSharedMemorySize, g->run_smem);
  }
  if (const char *v = getenv("FIBAR_WARM")) {
    g->warm = std::max(0, atoi(v));
    g->warm_set = true;
  }
  if (const char *v = getenv("FIBAR_DEBUG_WINDOW")) g->debug = atoi(v);
  if (const char *v = getenv("FIBAR_SERIAL")) g->serial = atoi(v) != 0;
  // The blur dataflow kernel runs in a CUDA green context of 48 SMs (5
  // blocks each, all resident): its polling lanes stop sharing SMs with the
  // next batch's front end.  With the round-2 front end the blur stage paces a
  // large batch, and 48 SMs beat 24 (config 2: 1091 -> 1176 Mev/s, config 5:
  // 1128 -> 1232; 40: 1161 / 1214, 56: 1194 / 1244, 64: 1045 / -).
  // FIBAR_GREEN=n sets the SM
  // count, 0 turns it off; without green-context support the blur stays on
  // the second stream with the whole GPU.
  int green_sms = 48;
  if (const char *v = getenv("FIBAR_GREEN")) green_sms = atoi(v);
  if (const char *v = getenv("FIBAR_ANCHOR_STREAM")) g->anchors_split = atoi(v) != 0;
  if (const char *v = getenv("FIBAR_STAGE_GRAPHS")) g->stage_graphs = atoi(v) != 0;
  if (const char *v = getenv("FIBAR_LONG_GRID")) g->long_grid_small = std::max(1, atoi(v));
  if (const char *v = getenv("FIBAR_GREEN_SMALL")) g->green_small = atoi(v) != 0;
  if (halo) green_sms = 0;
  if (green_sms > 0 && cfg->spatial_enabled && !g->serial) {
    const unsigned want = (unsigned)std::max(8, green_sms);
    CUdevice cdev;
    CUdevResource res, grp, rest;
    unsigned ng = 1;
    CUdevResourceDesc desc;
    const GreenApi &api = green_api();
    int cur = 0;
    cudaGetDevice(&cur);
    if (api.ok && api.deviceGet(&cdev, cur) == CUDA_SUCCESS &&
        api.getDevResource(cdev, &res, CU_DEV_RESOURCE_TYPE_SM) == CUDA_SUCCESS &&
        api.splitByCount(&grp, &ng, &res, &rest, 0, want) == CUDA_SUCCESS && ng == 1 &&
        api.generateDesc(&desc, &grp, 1) == CUDA_SUCCESS &&
        api.ctxCreate(&g->gctx, desc, cdev, CU_GREEN_CTX_DEFAULT_STREAM) == CUDA_SUCCESS) {
      CUstream cs;
      if (api.streamCreate(&cs, g->gctx, CU_STREAM_NON_BLOCKING, 0) == CUDA_SUCCESS) {
        g->gstream = (cudaStream_t)cs;
        int per = 5;   // all resident at 48 registers per thread (5 x 256 lanes per SM)
        if (const char *b = getenv("FIBAR_GREEN_BLOCKS")) per = std::max(1, atoi(b));
        g->gblocks = (int)grp.sm.smCount * per;
        cudaEventCreateWithFlags(&g->evP, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&g->evG, cudaEventDisableTiming);
      }
    }
    cudaGetLastError();
  }
  if (const char *v = getenv("FIBAR_PDL")) g->L.pdl = atoi(v) != 0;
  if (const char *v = getenv("FIBAR_TEMPORAL_ON_BLUR")) g->temporal_on_blur = atoi(v) != 0;
  g->full_graphs = !g->spatial;
  if (const char *v = getenv("FIBAR_FULL_GRAPHS")) g->full_graphs = atoi(v) != 0;
  {
    // contraction of the slower recurrence: events until any two float32
    // trajectories agree to the last bit, with a 1.6x margin
    const double r = std::max((double)cfg->alpha, (double)cfg->beta);
    const double steps = (r > 0.0 && r < 1.0) ? 24.0 * std::log(2.0) / -std::log(r) : 1024.0;
    g->twarm = (int)std::min(2048.0, std::max(64.0, std::ceil(1.6 * steps)));
  }
  // the window plus NPAR batches (the ingest of later batches writes their
  // ring keys while this batch's window pass still reads)
  g->R = 1LL << ceil_log2(n + 1 + NPAR * g->Bcap);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g->nsm, cudaDevAttrMultiProcessorCount, dev);
  {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_blur, TPB, 0);
    g->blur_grid_serial = g->nsm * std::max(1, std::min(per_sm, 4));   // graph form: nothing to overlap with
    // the blur stage overlaps the next batch's front end: one 256-thread block
    // per SM leaves the rest of each SM to the front end (measured: 1/SM gives
    // 10.2 ms per 10M config-2 events vs 11.2 at 2/SM and 12.6 serialised)
    const int occ = per_sm;
    per_sm = std::min(per_sm, g->serial ? 4 : 1);
    if (const char *v = getenv("FIBAR_BLUR_BLOCKS")) per_sm = std::min(occ, std::max(1, atoi(v)));
    g->blur_grid = g->nsm * std::max(1, per_sm);
    if (const char *v = getenv("FIBAR_BLUR_SLEEP")) g->blur_sleep = (unsigned)atoi(v);
    if (const char *v = getenv("FIBAR_GRAPHS")) g->graphs_on = atoi(v) != 0;
    if (const char *v = getenv("FIBAR_GRAPH_MAX")) g->graph_max = atoll(v);
    g->graph_max = std::min(g->graph_max, g->Bcap);
  }
  int rc = 0;
  const long long Bc = g->Bcap;
  const int nb_in = (int)((Bc + IN_TILE - 1) / IN_TILE);
  const int nb_rs = (int)((Bc + 2047) / 2048);
  const long long T = (Bc + CHUNK_MIN - 1) / CHUNK_MIN + 1;
  const long long npop_cap = Bc + n + 2;
  rc |= dalloc(&g->st, 1);
  rc |= dalloc(&g->pbar, n);
  rc |= dalloc(&g->l, n);
  for (int c = 0; c < 2; ++c) {
    rc |= dalloc(&g->sx[c], Bc);
    rc |= dalloc(&g->sy[c], Bc);
    rc |= dalloc(&g->sp_[c], Bc);
    if (cudaMallocHost((void **)&g->hx[c], sizeof(uint16_t) * Bc) != cudaSuccess ||
        cudaMallocHost((void **)&g->hy[c], sizeof(uint16_t) * Bc) != cudaSuccess ||
        cudaMallocHost((void **)&g->hp[c], sizeof(int8_t) * Bc) != cudaSuccess)
      rc |= fail(FIBAR_E_CUDA, "cudaMallocHost");
    cudaEventCreateWithFlags(&g->ev_h2d[c], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->ev_used[c], cudaEventDisableTiming);
  }
  cudaStreamCreateWithFlags(&g->cstream, cudaStreamNonBlocking);
  const int nsets = g->spatial ? NPAR : 1;
  for (int c = 0; c < nsets; ++c) rc |= dalloc(&g->blockcnt2[c], nb_in + 1);
  if (g->graphs_on && g->graph_max > 0) {
    for (int c = 0; c < nsets; ++c) {
      rc |= dalloc(&g->gx2[c], g->graph_max);
      rc |= dalloc(&g->gy2[c], g->graph_max);
      rc |= dalloc(&g->gp2[c], g->graph_max);
    }
  }
  for (int b = 0; b < NPAR; ++b) {
    if (b > 0 && !g->spatial) break;   // filter off: one batch at a time
    rc |= dalloc(&g->epol2[b], Bc);
    rc |= dalloc(&g->spol2[b], Bc);
  }
  for (int c = 0; c < (g->spatial ? NPAR : 1); ++c) rc |= dalloc(&g->longseg2[c], g->Bcap / LONG_SEG + 1);
  rc |= dalloc(&g->bsd, NPAR);
  if (!rc) cudaMemset(g->bsd, 0, NPAR * sizeof(BatchState));
  for (int c = 0; c < NPAR; ++c) {
    // the filter-off path runs every batch on one stream: one set suffices
    const bool own = c == 0 || g->spatial;
    if (own) {
      rc |= dalloc(&g->ekey2[c], Bc);
      rc |= dalloc(&g->ka2[c], Bc);
      rc |= dalloc(&g->va2[c], Bc);
      rc |= dalloc(&g->kb2[c], Bc);
      rc |= dalloc(&g->vb2[c], Bc);
    }
  }
  for (int c = 0; c < (g->spatial ? NPAR : 1); ++c) rc |= dalloc(&g->hist2[c], 1024LL * nb_rs + 1024LL * nb_rs / 4096 + 8);   // (digits of up to 10 bits)
  rc |= dalloc(&g->sel, 1);
  if (!rc) cudaMemset(g->sel, 0, sizeof(SelState));
  rc |= dalloc(&g->frame, n);
  if (g->use_gain) {
    rc |= dalloc(&g->gain, n);
    if (!rc) cudaMemcpy(g->gain, cfg->gain, sizeof(float) * n, cudaMemcpyHostToDevice);
  }
  if (g->spatial) {
    for (int c = 0; c < NPAR; ++c) {
      rc |= dalloc(&g->pt2[c], n);
      rc |= dalloc(&g->item2[c], npop_cap);
      rc |= dalloc(&g->t2_2[c], Bc);
      rc |= dalloc(&g->posrec2[c], Bc);
    }
    rc |= dalloc(&g->plast, n);
    rc |= dalloc(&g->wcnt, n);
    {
      // the blur stage is the latency-critical chain: its blocks go first when
      // SM slots free up, the next batch's front end fills the rest
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      if (const char *v = getenv("FIBAR_BLUR_PRIO")) hi = atoi(v) ? hi : lo;
      cudaStreamCreateWithPriority(&g->bstream, cudaStreamNonBlocking, hi);
    }
    cudaEventCreateWithFlags(&g->evT, cudaEventDisableTiming);
    for (int c = 0; c < NPAR; ++c) {
      cudaEventCreateWithFlags(&g->evF[c], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g->evB[c], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g->evBuf[c], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g->evS[c], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g->evA[c], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g->evV[c], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g->evN[c], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g->evR[c], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&g->evIn, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->evCp, cudaEventDisableTiming);
    {
      // the window part is the critical chain (latency-bound, small grids):
      // its blocks go first when SM slots free up (FIBAR_FRONT_PRIO=0: off)
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      int fp = hi;
      if (const char *v = getenv("FIBAR_FRONT_PRIO")) fp = atoi(v) ? hi : lo;
      cudaStreamCreateWithPriority(&g->fstream, cudaStreamNonBlocking, fp);
      // the eviction pass and the anchors run beside the chain: low priority
      int op = lo;
      if (const char *v = getenv("FIBAR_SIDE_PRIO")) op = atoi(v) ? hi : lo;
      cudaStreamCreateWithPriority(&g->pstream, cudaStreamNonBlocking, op);
      cudaStreamCreateWithPriority(&g->nstream, cudaStreamNonBlocking, op);
      cudaStreamCreateWithPriority(&g->astream, cudaStreamNonBlocking, lo);
      cudaStreamCreateWithPriority(&g->astream2, cudaStreamNonBlocking, lo);
      cudaStreamCreateWithPriority(&g->astream3, cudaStreamNonBlocking, lo);
      if (const char *v = getenv("FIBAR_SORT_LANES")) g->sort_lanes = std::min(3, std::max(1, atoi(v)));
      cudaStreamCreateWithPriority(&g->lstream, cudaStreamNonBlocking, lo);
      cudaStreamCreateWithPriority(&g->rstream, cudaStreamNonBlocking, lo);
      cudaStreamCreateWithPriority(&g->tstream, cudaStreamNonBlocking, hi);
      cudaEventCreateWithFlags(&g->evT0, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g->evT1, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g->evSnap, cudaEventDisableTiming);
      for (int c = 0; c < 2; ++c) {
        cudaEventCreateWithFlags(&g->evRd[c], cudaEventDisableTiming);
        rc |= dalloc(&g->snap[c], n);
      }
      if (const char *v = getenv("FIBAR_SNAP")) g->snap_on = atoi(v) != 0;
    }
    rc |= dalloc(&g->last_tile, g->n_tiles);
    for (int c = 0; c < NPAR; ++c) rc |= dalloc(&g->ptt2[c], g->n_tiles);
    rc |= dalloc(&g->rkey, g->R);
    rc |= dalloc(&g->rnext, g->R);
    for (int c = 0; c < NPAR; ++c) rc |= dalloc(&g->dp2[c], Bc);
    for (int c = 0; c < NPAR; ++c) {
      rc |= dalloc(&g->S2[c], Bc);
      rc |= dalloc(&g->Qt2[c], Bc);
      rc |= dalloc(&g->pmap2[c], npop_cap);
    }
    rc |= dalloc(&g->bv64, npop_cap);
    rc |= dalloc(&g->mv64, Bc);
    for (int c = 0; c < NPAR; ++c) {
      rc |= dalloc(&g->prep2[c], npop_cap);
      rc |= dalloc(&g->colist2[c], n + 1);
    }
    g->prep = g->prep2[0];
    for (int c = 0; c < NPAR; ++c) {
      rc |= dalloc(&g->anc3[c], (T + 1) * NCAND);
      rc |= dalloc(&g->anc23[c], (T + 1) * NFINE);
      rc |= dalloc(&g->anc03[c], T + 1);
      rc |= dalloc(&g->lc3[c], T + 1);
      rc |= dalloc(&g->lu3[c], T + 1);
    }
    rc |= dalloc(&g->ch, T);
    rc |= dalloc(&g->vl, 2 * T);   // the verifier's lists, by round parity
  }
  if (g->halo) {
    const long long nbh = (Bc + n + 2 + TPB - 1) / TPB;
    rc |= dalloc(&g->hslot, npop_cap);
    rc |= dalloc(&g->hlist, 4 * (Bc + n + 2));
    rc |= dalloc(&g->hcnt, 4 * nbh + 1);
  }
  if (g->spatial && getenv("FIBAR_DEBUG_TIMES")) {
    rc |= dalloc(&g->dbg_t, npop_cap);
    rc |= dalloc(&g->dbg_g, npop_cap);
  }
  if (rc) {
    fibar_destroy(g);
    return rc;
  }
  rc = init_state(g);
  if (rc) {
    fibar_destroy(g);
    return rc;
  }
  *out = g;
  return 0;
}

int fibar_destroy(fibar_engine *g) {
  if (!g) return 0;
  for (cudaStream_t st : {g->astream, g->astream2, g->astream3, g->lstream, g->nstream, g->fstream, g->pstream, g->bstream, g->rstream, g->tstream})
    if (st) cudaStreamSynchronize(st);
  void *ptrs[] = {g->st, g->pbar, g->l, g->gain, g->plast, g->wcnt, g->bsd, g->last_tile, g->rkey, g->rnext, g->raw_x,
                  g->raw_y, g->raw_p,
                  g->bv64, g->mv64, g->ch, g->vl, g->sel, g->frame,
                  g->cnt_tmp, g->tcnt_tmp, g->q_tmp, g->dbg_t, g->dbg_g, g->hslot, g->hlist, g->hcnt};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  for (cudaEvent_t ev : g->L.pool) cudaEventDestroy(ev);
  for (int c = 0; c < 2; ++c) {
    if (g->sx[c]) cudaFree(g->sx[c]);
    if (g->sy[c]) cudaFree(g->sy[c]);
    if (g->sp_[c]) cudaFree(g->sp_[c]);
    if (g->hx[c]) cudaFreeHost(g->hx[c]);
    if (g->hy[c]) cudaFreeHost(g->hy[c]);
    if (g->hp[c]) cudaFreeHost(g->hp[c]);
    if (g->ev_h2d[c]) cudaEventDestroy(g->ev_h2d[c]);
    if (g->ev_used[c]) cudaEventDestroy(g->ev_used[c]);
  }
  for (int c = 0; c < NPAR; ++c) {
    void *per[] = {g->pt2[c], g->ekey2[c], g->ka2[c], g->va2[c], g->kb2[c], g->vb2[c], g->item2[c], g->posrec2[c],
                   g->t2_2[c], g->ptt2[c], g->dp2[c], g->prep2[c], g->colist2[c], g->epol2[c], g->spol2[c],
                   g->S2[c], g->Qt2[c], g->pmap2[c], g->anc3[c], g->anc23[c], g->anc03[c], g->lc3[c], g->lu3[c]};
    for (void *p : per)
      if (p) cudaFree(p);
    for (cudaEvent_t ev : {g->evF[c], g->evB[c], g->evBuf[c], g->evA[c], g->evV[c], g->evN[c], g->evR[c], g->evS[c]})
      if (ev) cudaEventDestroy(ev);
  }
  if (g->cstream) cudaStreamDestroy(g->cstream);
  for (auto &ge : g->graphs)
    for (cudaGraphExec_t e : {ge.exec, ge.exec2, ge.exec3, ge.exec4, ge.exec5, ge.exec6})
      if (e) cudaGraphExecDestroy(e);
  if (g->capstream) cudaStreamDestroy(g->capstream);
  for (int c = 0; c < NPAR; ++c)
    for (void *q : {(void *)g->gx2[c], (void *)g->gy2[c], (void *)g->gp2[c], (void *)g->blockcnt2[c], (void *)g->hist2[c],
                    (void *)g->longseg2[c]})
      if (q) cudaFree(q);
  if (g->bstream) cudaStreamDestroy(g->bstream);
  for (void *q : {(void *)g->snap[0], (void *)g->snap[1]})
    if (q) cudaFree(q);
  for (cudaEvent_t ev : {g->evSnap, g->evRd[0], g->evRd[1], g->evT0, g->evT1})
    if (ev) cudaEventDestroy(ev);
  for (cudaStream_t st : {g->astream, g->astream2, g->astream3, g->lstream, g->rstream, g->tstream, g->nstream, g->fstream, g->pstream})
    if (st) cudaStreamDestroy(st);
  for (cudaEvent_t ev : {g->evIn, g->evCp})
    if (ev) cudaEventDestroy(ev);
  if (g->gstream) {
    cudaStreamSynchronize(g->gstream);
    cudaStreamDestroy(g->gstream);
  }
  if (g->gctx) green_api().ctxDestroy(g->gctx);
  for (cudaEvent_t ev : {g->evP, g->evG, g->evT})
    if (ev) cudaEventDestroy(ev);
  delete g;
  return 0;
}

int fibar_set_stream(fibar_engine *g, void *stream) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  g->L.stream = (cudaStream_t)stream;
  return 0;
}

int fibar_reset(fibar_engine *g) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  return init_state(g);
}

int fibar_process(fibar_engine *g, const uint16_t *x, const uint16_t *y, const int8_t *p, int64_t n, int32_t mem) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  if (g->halo) return fail(FIBAR_E_CONFIG, "halo-band engines take batches through fibar_halo_batch");
  if (n <= 0) return 0;
  long long off = 0;
  if (mem == FIBAR_MEM_DEVICE) {
    // contiguous device packets are coalesced without copies: the batch reads
    // them in place (the caller keeps them alive until the next flush point)
    if (g->hfill > 0) {
      int rc = launch_host_batch(g);
      if (rc) return rc;
    }
    while (off < n) {
      const bool contiguous = g->zn > 0 && x + off == g->zx + g->zn && y + off == g->zy + g->zn && p + off == g->zp + g->zn;
      if (g->zn > 0 && !contiguous) {
        // a packet elsewhere in memory: the pending in-place range and what
        // follows are gathered into the device staging set instead
        const long long zn = g->zn;
        g->zn = 0;
        gather_add(g, g->zx, g->zy, g->zp, zn);
      }
      if (g->dfill > 0) {
        const long long take = std::min((long long)n - off, g->Bcap - g->dfill);
        gather_add(g, x + off, y + off, p + off, take);
        off += take;
        if (g->dfill == g->Bcap || g->gt.n == GATHER_MAX) {
          int rc = flush_gather(g);
          if (rc) return rc;
        }
        continue;
      }
      if (g->zn == 0) {
        g->zx = x + off;
        g->zy = y + off;
        g->zp = p + off;
      }
      const long long take = std::min((long long)n - off, g->Bcap - g->zn);
      g->zn += take;
      off += take;
      if (g->zn == g->Bcap) {
        const long long zn = g->zn;
        g->zn = 0;
        int rc = run_batch_raw(g, g->zx, g->zy, g->zp, zn, nullptr);
        if (rc) return rc;
      }
    }
    return 0;
  }
  if (g->zn > 0 || g->dfill > 0) {
    int rc = run_batch(g);
    if (rc) return rc;
  }
  // large packets already in pinned memory are DMA'd straight into the device
  // staging set (no CPU copy); the call returns once those copies are done,
  // so the caller may reuse its buffers as with any host packet
  const long long dmin = direct_min(g);
  const bool direct = n - off >= dmin && is_pinned(x) && is_pinned(y) && is_pinned(p);
  cudaEvent_t last_direct = nullptr;
  if (direct && g->hfill > 0) {   // earlier staged packets go first
    int rc = launch_host_batch(g);
    if (rc) return rc;
  }
  while (direct && n - off >= dmin) {
    const int c = g->cur;
    const long long take = std::min((long long)n - off, g->Bcap);
    CK(cudaStreamWaitEvent(g->cstream, g->ev_used[c], 0));
    CK(cudaMemcpyAsync(g->sx[c], x + off, sizeof(uint16_t) * take, cudaMemcpyHostToDevice, g->cstream));
    CK(cudaMemcpyAsync(g->sy[c], y + off, sizeof(uint16_t) * take, cudaMemcpyHostToDevice, g->cstream));
    CK(cudaMemcpyAsync(g->sp_[c], p + off, sizeof(int8_t) * take, cudaMemcpyHostToDevice, g->cstream));
    CK(cudaEventRecord(g->ev_h2d[c], g->cstream));
    CK(cudaStreamWaitEvent(g->L.stream, g->ev_h2d[c], 0));
    last_direct = g->ev_h2d[c];
    g->cur ^= 1;
    off += take;
    int rc = run_batch_raw(g, g->sx[c], g->sy[c], g->sp_[c], take, g->ev_used[c]);
    if (rc) return rc;
  }
  if (last_direct) CK(cudaEventSynchronize(last_direct));
  while (off < n) {
    if (g->hfill == 0) CK(cudaEventSynchronize(g->ev_h2d[g->cur]));   // host set free again
    const long long take = std::min((long long)n - off, g->Bcap - g->hfill);
    memcpy(g->hx[g->cur] + g->hfill, x + off, sizeof(uint16_t) * take);
    memcpy(g->hy[g->cur] + g->hfill, y + off, sizeof(uint16_t) * take);
    memcpy(g->hp[g->cur] + g->hfill, p + off, sizeof(int8_t) * take);
    g->hfill += take;
    off += take;
    if (g->hfill == g->Bcap) {
      int rc = launch_host_batch(g);
      if (rc) return rc;
    }
  }
  return 0;
}

int fibar_halo_batch(fibar_engine *g, const uint16_t *x, const uint16_t *y, const int8_t *p, int64_t n, int32_t mem,
                     int64_t counts[4]) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  if (!g->halo) return fail(FIBAR_E_CONFIG, "not a halo-band engine");
  if (g->hopen) return fail(FIBAR_E_CONFIG, "previous halo batch not finished");
  if (n < 0 || n > g->Bcap) return fail(FIBAR_E_CONFIG, "halo batch larger than the batch capacity");
  int rc = sync_point(g);   // packets given to fibar_process run first
  if (rc) return rc;
  for (int c = 0; c < 4; ++c) g->hcount[c] = 0;
  if (n > 0) {
    cudaStream_t s = g->L.stream;
    if (mem != FIBAR_MEM_DEVICE) {
      CK(cudaMemcpyAsync(g->sx[0], x, sizeof(uint16_t) * n, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(g->sy[0], y, sizeof(uint16_t) * n, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(g->sp_[0], p, sizeof(int8_t) * n, cudaMemcpyHostToDevice, s));
      x = g->sx[0];
      y = g->sy[0];
      p = g->sp_[0];
    }
    const int par = (int)(g->batches % NPAR);
    rc = enqueue_batch(g, x, y, p, n, nullptr, par, false);
    if (rc) return rc;
    unsigned tot[5];
    for (int c = 0; c <= 4; ++c)
      CK(cudaMemcpyAsync(&tot[c], g->hcnt + (long long)c * g->hnb, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int c = 0; c < 4; ++c) g->hcount[c] = (long long)(tot[c + 1] - tot[c]);
    g->hopen = true;
  }
  for (int c = 0; c < 4; ++c) counts[c] = g->hcount[c];
  return 0;
}

int fibar_halo_round(fibar_engine *g, int32_t round, const uint64_t *in_words, uint64_t *out_words) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  if (!g->halo) return fail(FIBAR_E_CONFIG, "not a halo-band engine");
  if (!g->hopen) return 0;   // empty batch: nothing to blur
  Launcher &L = g->L;
  cudaStream_t s = L.stream;
  Ctx x = g->hctx;
  x.hin = (const unsigned long long *)in_words;
  if (round > 0) fibar_launch(L, "halo_epoch", k_halo_epoch, 1, 1, 0, s, x);
  fibar_launch(L, "blur", k_blur_halo, g->blur_grid_serial, TPB, 0, s, x);
  const long long n_in = g->hcount[0] + g->hcount[1], n_out = g->hcount[2] + g->hcount[3];
  if (n_out > 0)
    fibar_launch(L, "halo_collect", k_halo_collect, (int)((n_out + TPB - 1) / TPB), TPB, 0, s, x,
                 (const unsigned *)g->hlist, n_in, n_out, (unsigned long long *)out_words);
  CK(cudaGetLastError());
  return 0;
}

int fibar_halo_finish(fibar_engine *g) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  if (!g->halo) return fail(FIBAR_E_CONFIG, "not a halo-band engine");
  if (!g->hopen) return 0;
  fibar_launch(g->L, "final", k_final, g->nsm * 8, TPB, 0, g->L.stream, g->hctx);
  CK(cudaGetLastError());
  g->hopen = false;
  g->batches++;
  return 0;
}

int fibar_flush(fibar_engine *g) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  return sync_point(g);
}

int fibar_pending(fibar_engine *g, int64_t *device_events, int64_t *staged_events) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  if (device_events) *device_events = g->zn + g->dfill;   // device packets still read from where they are
  if (staged_events) *staged_events = g->hfill;
  return 0;
}

int fibar_render(fibar_engine *g, int32_t mode, double fixed_bound, uint8_t *out, int32_t out_mem, double *bounds,
                 int32_t *degenerate) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  int rc = sync_point(g);
  if (rc) return rc;
  return render_core(g->L, g->l, g->n_pix, mode, fixed_bound, out, out_mem, bounds, degenerate, g->sel, g->frame, g->nsm);
}

int fibar_render_async(fibar_engine *g, int32_t mode, double fixed_bound, uint8_t *out, int32_t out_mem, void *meta,
                       void *ready) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  if (!meta || !ready) return fail(FIBAR_E_CONFIG, "render_async needs meta and an event");
  int rc = run_batch(g);
  if (rc) return rc;
  Launcher &L = g->L;
  cudaStream_t s0 = L.stream;
  const bool on_blur = g->spatial && g->last_b >= 0 && !g->serial;
  // after the newest blur stage, on its stream: the next batch's front end
  // (engine stream) does not wait for the read-out, its temporal replay does
  // -- unless the read-out works on a snapshot (rstream): then the blur
  // stream only carries the snapshot copy
  const bool snap = on_blur && g->snap_on && g->rstream && g->snap[0];
  cudaStream_t rs = on_blur ? g->bstream : s0;
  const float *src = g->l;
  if (snap) {
    const int i = (int)(g->n_snap++ & 1);
    if (g->rd_used[i]) CK(cudaStreamWaitEvent(g->bstream, g->evRd[i], 0));   // its previous read-out is done
    L.stream = g->bstream;
    fibar_launch(L, "snap", k_snap, g->nsm * 2, TPB, 0, g->bstream, (const float *)g->l, g->snap[i], g->n_pix);
    CK(cudaEventRecord(g->evSnap, g->bstream));
    CK(cudaStreamWaitEvent(g->rstream, g->evSnap, 0));
    rs = g->rstream;
    src = g->snap[i];
  }
  L.stream = rs;
  // rendered into device memory (render_core would wait for a host frame),
  // copied to a host frame asynchronously here
  const bool dev_out = out_mem == FIBAR_MEM_DEVICE;
  rc = render_core(L, src, g->n_pix, mode, fixed_bound, dev_out ? out : g->frame, FIBAR_MEM_DEVICE, nullptr, nullptr,
                   g->sel, g->frame, g->nsm);
  if (!rc && !dev_out) {
    cudaError_t e = cudaMemcpyAsync(out, g->frame, g->n_pix, cudaMemcpyDeviceToHost, rs);
    if (e != cudaSuccess) rc = cuda_fail(e, "render_async frame");
  }
  if (!rc) {
    const cudaMemcpyKind kind = dev_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    cudaError_t e = cudaMemcpyAsync(meta, &g->sel->lo, 2 * sizeof(double) + sizeof(int), kind, rs);
    if (e != cudaSuccess) rc = cuda_fail(e, "render_async meta");
  }
  if (!rc && on_blur) {
    g->mark(8, rs);   // 8: read-out end
    cudaError_t e = cudaEventRecord(g->evB[g->last_b], rs);   // later batches order after the read-out
    if (e != cudaSuccess) rc = cuda_fail(e, "render_async event");
    if (!rc && snap) {
      const int i = (int)((g->n_snap - 1) & 1);
      e = cudaEventRecord(g->evRd[i], rs);
      if (e != cudaSuccess) rc = cuda_fail(e, "render_async event");
      g->rd_used[i] = true;
    }
  }
  if (!rc) {
    cudaError_t e = cudaEventRecord((cudaEvent_t)ready, rs);
    if (e != cudaSuccess) rc = cuda_fail(e, "render_async ready");
  }
  L.stream = s0;
  return rc;
}

int fibar_render_grid(const float *l_dev, int64_t n, int32_t mode, double fixed_bound, uint8_t *out, int32_t out_mem,
                      double *bounds, int32_t *degenerate, void *stream) {
  // read-out scratch per device, one caller at a time (the scratch is shared
  // by every stream of that device)
  struct Scratch {
    SelState *sel = nullptr;
    uint8_t *frame = nullptr;
    long long cap = 0;
    int nsm = 0;
  };
  static Scratch per_dev[64];
  static std::mutex mu;
  if (!l_dev || n < 1) return fail(FIBAR_E_CONFIG, "empty grid");
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(FIBAR_E_CONFIG, "device index out of range");
  std::lock_guard<std::mutex> lock(mu);
  Scratch &sc = per_dev[dev];
  if (!sc.sel) {
    int rc = dalloc(&sc.sel, 1);
    if (rc) return rc;
    CK(cudaMemset(sc.sel, 0, sizeof(SelState)));
    cudaDeviceGetAttribute(&sc.nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  if (out_mem != FIBAR_MEM_DEVICE && n > sc.cap) {
    if (sc.frame) cudaFree(sc.frame);
    sc.frame = nullptr;
    int rc = dalloc(&sc.frame, n);
    if (rc) return rc;
    sc.cap = n;
  }
  Launcher L;
  L.stream = (cudaStream_t)stream;
  int rc = render_core(L, l_dev, n, mode, fixed_bound, out, out_mem, bounds, degenerate, sc.sel, sc.frame, sc.nsm);
  if (!rc && !(bounds || degenerate || out_mem != FIBAR_MEM_DEVICE))
    CK(cudaStreamSynchronize(L.stream));   // the scratch is reused by the next caller
  return rc;
}

int fibar_read_qs(fibar_engine *g, int64_t qs[10]) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  int rc = sync_point(g);
  if (rc) return rc;
  DevState h;
  CK(cudaMemcpyAsync(&h, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, g->L.stream));
  CK(cudaStreamSynchronize(g->L.stream));
  qs[0] = h.s % (g->n_pix + 1);
  qs[1] = h.E - h.s;
  qs[2] = h.q;
  qs[3] = h.npix;
  qs[4] = h.ntiles;
  qs[5] = h.blur;
  qs[6] = h.stale;
  qs[7] = h.qtmin;
  qs[8] = h.qtmax;
  qs[9] = h.evctr;
  if (!g->spatial) {
    qs[0] = 0;
    qs[1] = 0;
  }
  return 0;
}

int fibar_debug_stale_items(fibar_engine *g, int64_t *event_idx, uint32_t *pixel, int64_t cap, int64_t *n_out) {
  if (!g || !n_out) return fail(FIBAR_E_CONFIG, "null argument");
  int rc = sync_point(g);
  if (rc) return rc;
  *n_out = 0;
  if (!g->spatial || g->last_par < 0) return 0;
  const int par = g->last_par;
  BatchState bs;
  CK(cudaMemcpyAsync(&bs, g->bsd + par, sizeof(BatchState), cudaMemcpyDeviceToHost, g->L.stream));
  CK(cudaStreamSynchronize(g->L.stream));
  if (bs.npop <= 0) return 0;
  std::vector<Item> items((size_t)bs.npop);
  CK(cudaMemcpyAsync(items.data(), g->item2[par], sizeof(Item) * (size_t)bs.npop, cudaMemcpyDeviceToHost,
                     g->L.stream));
  CK(cudaStreamSynchronize(g->L.stream));
  long long k = 0;
  for (const Item &it : items) {
    if (it.pix == FIBAR_NONE) continue;
    if (k < cap) {
      if (event_idx) event_idx[k] = bs.E0 + (long long)it.jrel;
      if (pixel) pixel[k] = it.pix;
    }
    ++k;
  }
  *n_out = k;
  return k > cap ? fail(FIBAR_E_CONFIG, "stale item buffer too small") : 0;
}

int fibar_debug_regulate(int64_t num, int64_t den, int32_t tile_area, int64_t q_min, int64_t q_max, const uint32_t *len,
                         const uint32_t *np, const uint32_t *nt, int64_t n, uint32_t *out_fast, uint32_t *out_exact) {
  if (n <= 0) return 0;
  const long long numA = num * (long long)tile_area;
  if (!(numA > 0 && numA < (1LL << 24) && den > 0 && den < (1LL << 24) && q_min >= 1 && q_min <= q_max && q_max < (1LL << 22) &&
        den * (q_max + 2) < (1LL << 29)))
    return fail(FIBAR_E_CONFIG, "regulate32x does not apply to these parameters");
  Ctx x{};
  x.num = num;
  x.den = den;
  x.A = tile_area;
  x.numA = numA;
  x.qmin = q_min;
  x.qmax = q_max;
  unsigned *d = nullptr;
  CK(cudaMalloc(&d, sizeof(unsigned) * 5 * n));
  cudaError_t e = cudaMemcpy(d, len, sizeof(unsigned) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d + n, np, sizeof(unsigned) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d + 2 * n, nt, sizeof(unsigned) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    k_debug_regulate<<<(int)std::min<long long>(1184, (n + TPB - 1) / TPB), TPB>>>(x, d, d + n, d + 2 * n, (long long)n, d + 3 * n,
                                                                                  d + 4 * n);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out_fast, d + 3 * n, sizeof(unsigned) * n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(out_exact, d + 4 * n, sizeof(unsigned) * n, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "fibar_debug_regulate");
  return 0;
}

int fibar_debug_trace(fibar_engine *g, int64_t cap, int64_t *batch, int32_t *label, double *ms, int64_t *n_out) {
  if (!g || !n_out) return fail(FIBAR_E_CONFIG, "null argument");
  CK(cudaDeviceSynchronize());
  const long long n = (long long)g->tr.size();
  *n_out = n;
  for (long long i = 0; i < n && i < cap; ++i) {
    float t = 0.f;
    cudaEventElapsedTime(&t, g->tr[0].ev, g->tr[i].ev);
    batch[i] = g->tr[i].batch;
    label[i] = g->tr[i].label;
    ms[i] = t;
  }
  for (auto &r : g->tr) cudaEventDestroy(r.ev);
  g->tr.clear();
  cudaGetLastError();
  return 0;
}

int fibar_counters(fibar_engine *g, int64_t *event_count, int64_t *oob_dropped) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  int rc = sync_point(g);
  if (rc) return rc;
  DevState h;
  CK(cudaMemcpyAsync(&h, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, g->L.stream));
  CK(cudaStreamSynchronize(g->L.stream));
  if (event_count) *event_count = h.E;
  if (oob_dropped) *oob_dropped = h.oob;
  return 0;
}

int fibar_read_state(fibar_engine *g, float *p_bar, float *l, uint16_t *active, uint8_t *tiles, uint16_t *qx,
                     uint16_t *qy) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  int rc = sync_point(g);
  if (rc) return rc;
  cudaStream_t s = g->L.stream;
  const long long n = g->n_pix;
  if (p_bar) CK(cudaMemcpyAsync(p_bar, g->pbar, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
  if (l) CK(cudaMemcpyAsync(l, g->l, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
  if (active || tiles || qx || qy) {
    if (!g->cnt_tmp) {
      rc |= dalloc(&g->cnt_tmp, n);
      rc |= dalloc(&g->tcnt_tmp, g->n_tiles);
      rc |= dalloc(&g->q_tmp, 2 * (n + 1));
      if (rc) return rc;
    }
    CK(cudaMemsetAsync(g->cnt_tmp, 0, sizeof(unsigned) * n, s));
    CK(cudaMemsetAsync(g->tcnt_tmp, 0, sizeof(unsigned) * g->n_tiles, s));
    Ctx x = g->ctx(nullptr, nullptr, 0, 0);
    if (g->spatial) {
      fibar_launch(g->L, "state_active", k_active_counts, g->nsm * 4, TPB, 0, s, x, g->cnt_tmp);
      fibar_launch(g->L, "state_tiles", k_tile_counts, g->nsm * 4, TPB, 0, s, x, g->cnt_tmp, g->tcnt_tmp);
      fibar_launch(g->L, "state_ring", k_ring_xy, g->nsm * 4, TPB, 0, s, x, g->q_tmp, g->q_tmp + n + 1);
    } else {
      CK(cudaMemsetAsync(g->q_tmp, 0, sizeof(uint16_t) * 2 * (n + 1), s));
    }
    CK(cudaGetLastError());
    std::vector<unsigned> hc, ht;
    if (active) hc.resize(n);
    if (tiles) ht.resize(g->n_tiles);
    if (active) CK(cudaMemcpyAsync(hc.data(), g->cnt_tmp, sizeof(unsigned) * n, cudaMemcpyDeviceToHost, s));
    if (tiles) CK(cudaMemcpyAsync(ht.data(), g->tcnt_tmp, sizeof(unsigned) * g->n_tiles, cudaMemcpyDeviceToHost, s));
    if (qx) CK(cudaMemcpyAsync(qx, g->q_tmp, sizeof(uint16_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    if (qy) CK(cudaMemcpyAsync(qy, g->q_tmp + n + 1, sizeof(uint16_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (active)
      for (long long i = 0; i < n; ++i) active[i] = (uint16_t)std::min<unsigned>(hc[i], 65535u);
    if (tiles)
      for (long long i = 0; i < g->n_tiles; ++i) tiles[i] = (uint8_t)std::min<unsigned>(ht[i], 255u);
  }
  CK(cudaStreamSynchronize(s));
  return 0;
}

int fibar_stats(fibar_engine *g, int64_t stats[16]) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  int rc = sync_point(g);
  if (rc) return rc;
  DevState h;
  CK(cudaMemcpyAsync(&h, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, g->L.stream));
  CK(cudaStreamSynchronize(g->L.stream));
  stats[0] = g->L.launches;
  stats[1] = g->batches;
  stats[2] = h.chunks;
  stats[3] = h.mismatch;
  stats[4] = h.pops;
  // tile_count (u8) can only saturate when a tile has more than 255 pixels
  stats[5] = h.saturated + ((g->spatial && g->A > 255 && h.E > 0) ? 1 : 0);
  stats[6] = h.E;
  stats[7] = g->Bcap;
  stats[8] = h.warm_pops;
  stats[9] = h.coop_iters;
  stats[10] = h.fix_rounds;
  stats[11] = h.dbg_bad;
  return 0;
}

int fibar_profile(fibar_engine *g, int32_t enable) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  join_blur(g);
  CK(cudaStreamSynchronize(g->L.stream));
  g->L.prof = enable != 0;
  g->L.recs.clear();
  g->L.used = 0;
  return 0;
}

int fibar_profile_read(fibar_engine *g, int32_t max_entries, char *names, int32_t name_len, double *total_ms,
                       int64_t *launches, int32_t *n_entries) {
  if (!g) return fail(FIBAR_E_CONFIG, "null engine");
  join_blur(g);
  CK(cudaStreamSynchronize(g->L.stream));
  std::vector<std::string> keys;
  std::vector<double> ms;
  std::vector<long long> cnt;
  for (auto &r : g->L.recs) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, r.a, r.b));
    size_t k = 0;
    for (; k < keys.size(); ++k)
      if (keys[k] == r.name) break;
    if (k == keys.size()) {
      keys.push_back(r.name);
      ms.push_back(0.0);
      cnt.push_back(0);
    }
    ms[k] += t;
    cnt[k] += 1;
  }
  const int m = (int)std::min<size_t>(keys.size(), (size_t)max_entries);
  for (int k = 0; k < m; ++k) {
    strncpy(names + (size_t)k * name_len, keys[k].c_str(), name_len - 1);
    names[(size_t)k * name_len + name_len - 1] = 0;
    total_ms[k] = ms[k];
    launches[k] = cnt[k];
  }
  *n_entries = m;
  g->L.recs.clear();
  g->L.used = 0;
  return 0;
}

// debug: item completion / grab timestamps (ns) of the last batch; FIBAR_DEBUG_TIMES must be set
int fibar_debug_times(fibar_engine *g, uint64_t *done_ns, uint64_t *grab_ns, int64_t n) {
  if (!g || !g->dbg_t) return fail(FIBAR_E_CONFIG, "debug timestamps not enabled");
  join_blur(g);
  CK(cudaStreamSynchronize(g->L.stream));
  CK(cudaMemcpy(done_ns, g->dbg_t, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(grab_ns, g->dbg_g, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  return 0;
}

// debug: copy the blur prep records (80 B each) of the last batch
int fibar_debug_prep(fibar_engine *g, void *out, int64_t n) {
  if (!g || !g->prep) return fail(FIBAR_E_CONFIG, "no prep");
  join_blur(g);
  CK(cudaStreamSynchronize(g->L.stream));
  CK(cudaMemcpy(out, g->prep, sizeof(BlurPrep) * n, cudaMemcpyDeviceToHost));
  return 0;
}

int fibar_debug_readout_times(fibar_engine *g, uint64_t ts[16]) {
  if (!g || !ts) return fail(FIBAR_E_CONFIG, "null argument");
  join_blur(g);
  CK(cudaStreamSynchronize(g->L.stream));
  CK(cudaMemcpy(ts, g->sel->ts, sizeof(uint64_t) * 16, cudaMemcpyDeviceToHost));
  return 0;
}

int fibar_decode_evf1(const uint8_t *records, int64_t nrec, int32_t width, int32_t height, uint64_t t_base,
                      uint16_t *x, uint16_t *y, int8_t *p, uint64_t *t, int64_t *first_bad, void *stream) {
  if (nrec < 0 || !first_bad) return fail(FIBAR_E_CONFIG, "bad arguments");
  *first_bad = -1;
  if (nrec == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = (int)((nrec + EV_TILE - 1) / EV_TILE);
  unsigned *dt = nullptr;
  unsigned long long *bsum = nullptr, *bad = nullptr;
  CK(cudaMallocAsync((void **)&dt, sizeof(unsigned) * nrec, s));
  CK(cudaMallocAsync((void **)&bsum, sizeof(unsigned long long) * (nb + 1), s));
  CK(cudaMallocAsync((void **)&bad, sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), s));
  k_evf1_decode<<<nb, TPB, 0, s>>>(reinterpret_cast<const uint4 *>(records), reinterpret_cast<const uint2 *>(records),
                                   nrec, width, height, x, y, p, dt, bsum, bad);
  k_evf1_block_scan<<<1, 1024, 0, s>>>(bsum, nb, (unsigned long long)t_base);
  if (t) k_evf1_times<<<nb, TPB, 0, s>>>(dt, nrec, bsum, reinterpret_cast<unsigned long long *>(t));
  unsigned long long hb = 0;
  CK(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, s));
  cudaFreeAsync(dt, s);
  cudaFreeAsync(bsum, s);
  cudaFreeAsync(bad, s);
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  *first_bad = hb == ~0ull ? -1 : (int64_t)hb;
  return 0;
}

int fibar_copy_brightness(fibar_engine *g, float *dst, int32_t dst_mem) {
  if (!g || !dst) return fail(FIBAR_E_CONFIG, "null argument");
  int rc = sync_point(g);
  if (rc) return rc;
  CK(cudaMemcpyAsync(dst, g->l, sizeof(float) * g->n_pix,
                     dst_mem == FIBAR_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, g->L.stream));
  if (dst_mem != FIBAR_MEM_DEVICE) CK(cudaStreamSynchronize(g->L.stream));
  return 0;
}

int fibar_brightness_ptr(fibar_engine *g, float **out) {
  if (!g || !out) return fail(FIBAR_E_CONFIG, "null argument");
  int rc = sync_point(g);
  if (rc) return rc;
  *out = g->l;
  return 0;
}

}  // extern "C"
