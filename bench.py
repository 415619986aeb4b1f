"""Benchmark of the FIBAR reconstruction hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 3]

Headline workload (BASELINE.json configs[2], the largest single-GPU config):
config 3 -- 1280x720 sensor, 100M events of the seeded moving-texture stream
plus 20 % noise and Zipf hot pixels (paper_2510_20071_b200/workloads.py),
spatial filter ON, 100k-event packets, a robust read-out after EVERY packet.
One *step* = reset the engine, push all 1,000 packets through
``ReconstructionEngine.process_array`` and render a frame after each one.

* ``value``: packets already resident in HBM (one separately allocated
  DeviceEventArray per packet), frames left in HBM; per-step CUDA events on the
  engine stream, L2 flushed (256 MiB write) between steps, max over ranks.
* ``e2e``: the same step through the reference's own frame loop ``run()`` with
  host packets (numpy views of pinned memory: H2D inside the timed region) and
  every frame copied back to the host.
* ``parity``: outside the timed region the device arm runs once more keeping
  all 1,000 frames in HBM; their hashes and the final reference-layout state
  (p_bar, l, active_count, tile_count, ring, qs) must equal the C oracle's on
  the same stream (the ``cpu_baseline`` leg).  A mismatch fails the run.
* ``roofline``: the dominant kernel by serialised device time (a profiled step
  on an engine built with FIBAR_SERIAL=1 FIBAR_PDL=0, per-kernel CUDA events),
  its SURVEY 8(d) algorithmic bytes per launch over its mean launch time,
  against MEASURED_PEAKS.json hbm_gbs.  ``path_roofline`` applies 8(d)'s
  per-event model (B_ON / B_OFF) to the whole step.
* ``filter_off``: the filter-OFF rows of the metric -- config 4's stream at
  1M-event packets with a read-out per packet, and config 1 -- each device
  timed and checked against the oracle's final state.
* ``cpu_baseline``: the C oracle (a restatement of the reference's numba
  kernels, single thread like the reference) on the same 100M-event stream at
  the same read-out cadence.

``--impl reference`` times that CPU implementation alone (rank 0; other ranks
exit) and prints the same JSON shape with ``"impl": "reference"``.
Multi-GPU: filter OFF runs row bands (strong scaling).  Filter
ON runs the halo row bands (exact, NCCL halo exchange, strong scaling);
``--replicas`` runs N independent streams instead (weak scaling, no collective).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import sys
import threading
import time
from fractions import Fraction

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2510_20071_b200 import workloads  # noqa: E402
from paper_2510_20071_b200.core import SensorGeometry, compute_params  # noqa: E402

METRIC = "Mevents/s reconstructed (spatial filter on/off) at 1/2/4/8 B200; % HBM roofline"
UNIT = "Mevents/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--events", type=int, default=None, help="override the config's event count")
    ap.add_argument("--packet", type=int, default=None)
    ap.add_argument("--filter", default=None, choices=("on", "off"))
    ap.add_argument("--batch-cap", type=int, default=0, help="device batch capacity (0: the engine's default)")
    ap.add_argument("--readout", default=None, choices=("end", "packet"),
                    help="robust read-out at the end of the stream or after every packet (config default)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle leg (and with it the parity check)")
    ap.add_argument("--no-off", action="store_true", help="skip the filter-OFF extra lines")
    ap.add_argument("--profile-only", action="store_true", help="one step, for ncu launch lists")
    ap.add_argument("--bands", action="store_true", help="row bands on one rank (filter ON: halo bands)")
    ap.add_argument("--replicas", action="store_true", help="N>1, filter ON: N independent streams, no collective")
    ap.add_argument("--halo", type=int, default=16, help="halo rows of the filter-ON row bands")
    ap.add_argument("--halo-batch", type=int, default=1 << 20, help="events per halo-band batch")
    return ap.parse_args()


def workload(args, rank, config=None, events=None, packet=None, spatial=None, readout=None):
    cfg = workloads.CONFIGS[config or args.config]
    geom = cfg["geometry"]
    n = events or (args.events if config is None else None) or cfg["n"]
    if spatial is None:
        spatial = cfg["spatial"] if cfg["spatial"] is not None else True
        if args.filter and config is None:
            spatial = args.filter == "on"
    packet = packet or (args.packet if config is None else None) or cfg["packet"] or 100_000
    kw = {"speed": cfg["speed"]} if "speed" in cfg else {}
    ev = workloads.make_cached(cfg["kind"], geom, n, seed=rank, **kw)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=spatial)
    if readout is None:
        readout = (args.readout if config is None else None) or cfg.get("readout", "end")
    if config is None:
        args.readout = readout
    ro = "robust read-out after every packet" if readout == "packet" else "robust read-out at end"
    name = f"config{config or args.config}:{geom.width}x{geom.height},{n / 1e6:g}M events,{cfg['kind']}," \
           f"filter {'on' if spatial else 'off'},{packet}-event packets,{ro}"
    return geom, params, ev, packet, name


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling via NVML during the timed region."""

    def __init__(self, index=0, period=float(os.environ.get("BENCH_CLOCK_PERIOD", "0.05"))):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# SURVEY 8(d) algorithmic bytes per launch of each kernel, from the batch
# statistics (B events, P evictions, D distinct pixels, NB blurs) -- the bytes
# the kernel's job must read and write once:
#   window_run / window_fix / anchor*: 8 B per event (the two 4-byte link
#       distances) + 8 B per eviction (the evicted entry's next-event links)
#   blur: 8 B per blur (centre read + write; taps on-chip)
#   temporal_runs / temporal_long: 5 B per event (x, y, p) + 16 B per
#       distinct pixel (p_bar and l read + written)
#   readout: 9 B per pixel (robust: one selection pass + read + u8 write)
#   rs_scatter: 16 B per event (key + index in and out); rs_hist 4 B per event
#   popj: 4 B per event + 12 B per eviction; link: 24 B per event
#   count_inb 4 B, compact 18 B per event (x, y, p in; keys, ring key out)
def kernel_bytes(name, B, P, D, NB, n_pix):
    table = {
        "window_run": 8 * B + 8 * P, "window_fix": 8 * B + 8 * P, "anchor": 8 * B, "anchor2": 8 * B,
        "blur": 8 * NB, "temporal": 5 * B + 16 * D, "temporal_long": 5 * B + 16 * D,
        "readout": 9 * n_pix, "rs_scatter": 16 * B, "rs_hist": 4 * B, "popj": 4 * B + 12 * P, "link": 24 * B,
        "count_inb": 4 * B, "compact": 18 * B,
    }
    return table.get(name)


def workload_class(name: str) -> str:
    """The workload string without its event count: per-launch traffic of a
    device batch does not depend on how long the stream is."""
    parts = name.split(",")
    return ",".join(p for p in parts if not p.endswith("M events"))


def committed_traffic(kernel: str, workload_name: str, batch_cap: int):
    """DRAM bytes per launch of `kernel` from the latest committed ncu --set full
    capture (profiles/*_traffic.json, written by scripts/summarize_ncu.py) --
    only when that capture was taken on this workload class and device batch."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    for f in reversed(files):
        try:
            d = json.load(open(f))
        except (OSError, ValueError):
            continue
        if d.get("workload_class") != workload_class(workload_name) or d.get("device_batch_cap") != batch_cap:
            continue
        v = d.get("bytes_per_launch", {}).get(kernel)
        if v:
            return v, os.path.basename(f)
    return None, None


def frame_hash(px) -> str:
    return hashlib.sha256(np.ascontiguousarray(px).tobytes()).hexdigest()[:16]


def state_digest(d) -> str:
    h = hashlib.sha256()
    for k in ("p_bar", "l", "active_count", "tile_count", "qx", "qy", "qs"):
        h.update(np.ascontiguousarray(d[k]).tobytes())
    return h.hexdigest()


def separate_device_packets(ev, cuts, dev):
    """One separately allocated DeviceEventArray per packet (a real device
    stream: packets are not views of one buffer)."""
    import torch
    from paper_2510_20071_b200.pipeline import DeviceEventArray
    out = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        out.append(DeviceEventArray(torch.from_numpy(ev.x[a:b].view(np.int16)).to(dev),
                                    torch.from_numpy(ev.y[a:b].view(np.int16)).to(dev),
                                    torch.from_numpy(ev.p[a:b]).to(dev)))
    return out


def device_timer(dev, stream, dist, flush_buf):
    import torch

    def timed(step, steps, warmup):
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        total = 0.0
        for _ in range(steps):
            flush_buf.zero_()
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step()
            s1.record(stream)
            torch.cuda.synchronize()
            total += s0.elapsed_time(s1) / 1e3
        if dist:
            t = torch.tensor([total], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total = float(t.item())
        return total
    return timed


def profiled_engine(geom, params, batch_cap):
    """An engine with the serial schedule and no programmatic dependent launch,
    so per-kernel CUDA events measure each kernel alone (DESIGN.md §9 knobs are
    read at construction)."""
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    saved = {k: os.environ.get(k) for k in ("FIBAR_SERIAL", "FIBAR_PDL")}
    os.environ.update(FIBAR_SERIAL="1", FIBAR_PDL="0")
    try:
        return ReconstructionEngine(geom, params, batch_capacity=batch_cap)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def run_ours(args, rank, world, dist):
    import torch
    from paper_2510_20071_b200.core import EventArray
    from paper_2510_20071_b200.pipeline import ReconstructionEngine, run

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    geom, params, ev, packet, name = workload(args, rank)
    n = len(ev)
    eng = ReconstructionEngine(geom, params, batch_capacity=args.batch_cap)
    args.batch_cap = eng._bcap   # the effective device batch capacity
    stream = torch.cuda.current_stream(dev)
    frame = torch.empty((geom.height, geom.width), dtype=torch.uint8, device=dev)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    cuts = list(range(0, n, packet)) + [n]
    dev_packets = separate_device_packets(ev, cuts, dev)
    per_packet = args.readout == "packet"
    meta_dev = torch.empty(4, dtype=torch.float64, device=dev)
    timed = device_timer(dev, stream, dist, flush_buf)

    def step_device(engine=eng, frames=None):
        engine.reset()
        if per_packet:
            # a read-out after every packet, enqueued asynchronously behind the
            # packet's blur stage (the next packet's front end overlaps it);
            # the step ends when the last frame is in HBM
            af = None
            for k, blk in enumerate(dev_packets):
                engine.process_array(blk)
                af = engine.render_async("robust", out=frame if frames is None else frames[k], meta=meta_dev)
            stream.wait_event(af.event)
            return
        for blk in dev_packets:
            engine.process_array(blk)
        engine.render_device("robust", out=frame if frames is None else frames[0])

    if args.profile_only:
        step_device()
        torch.cuda.synchronize()
        print(json.dumps({"workload_class": workload_class(name), "device_batch_cap": args.batch_cap,
                          "batches": eng.stats()["batches"]}))
        return None

    # host arm: pinned host columns, numpy views per packet
    xh = torch.from_numpy(ev.x.view(np.int16)).pin_memory().numpy().view(np.uint16)
    yh = torch.from_numpy(ev.y.view(np.int16)).pin_memory().numpy().view(np.uint16)
    ph = torch.from_numpy(ev.p).pin_memory().numpy()
    host_packets = [EventArray(ev.t[a:b], xh[a:b], yh[a:b], ph[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    last_frame = {}
    # per-packet read-outs go through the reference's own frame loop, run()
    # (frames at each packet's end time, delivered to the host)
    pp_times = [int(ev.t[b - 1]) + 1 for b in cuts[1:]]

    def step_host():
        eng.reset()
        if per_packet:
            run(eng, host_packets, readout_times=pp_times, frame_sink=lambda k, f: last_frame.__setitem__("f", f))
            return
        for blk in host_packets:
            eng.process_array(blk)
        last_frame["f"] = eng.render("robust")

    l0 = eng.stats()["launches"]
    with ClockSampler(dev.index) as clk:
        t_dev = timed(step_device, args.steps, args.warmup)
    launches = (eng.stats()["launches"] - l0) // (args.steps + args.warmup)
    value = n * world * args.steps / t_dev / 1e6
    ms_per_step = t_dev / args.steps * 1e3

    # parity run (untimed): every frame kept in HBM, hashed, plus the final state
    nfr = len(dev_packets) if per_packet else 1
    frames_all = torch.empty((nfr, geom.height, geom.width), dtype=torch.uint8, device=dev)
    b0 = eng.stats()["batches"]   # a host-side count (reset() clears only the device counters)
    step_device(frames=frames_all)
    torch.cuda.synchronize()
    st1 = eng.stats()
    fr_host = frames_all.cpu().numpy()
    gpu_hashes = [frame_hash(f) for f in fr_host]
    del frames_all, fr_host
    gpu_state = eng.state_arrays()
    gpu_digest = state_digest(gpu_state)
    qs = gpu_state["qs"]
    blurs = int(qs[5])
    b_batches = max(1, st1["batches"] - b0)
    pops = st1["pops"]
    pid = ev.y.astype(np.int64) * geom.width + ev.x
    u_packet = float(np.mean([np.unique(pid[a:a + packet]).size / min(packet, n - a)
                              for a in range(0, min(n, 50 * packet), packet)]))
    B_mean = n / b_batches
    D_mean = float(np.mean([np.unique(pid[a:a + int(B_mean)]).size for a in range(0, min(n, 20 * int(B_mean)), int(B_mean))]))

    # per-kernel serialised device time (untimed profiled step, own engine)
    peng = profiled_engine(geom, params, args.batch_cap)
    peng.profile(True)
    step_device(engine=peng)
    prof = peng.profile_read()
    peng.profile(False)
    peng.close()
    tot_ms = sum(v[0] for v in prof.values())
    dname, (dms, dcnt) = max(prof.items(), key=lambda kv: kv[1][0])
    P_mean = pops / b_batches
    NB_mean = blurs / b_batches
    bytes_launch = kernel_bytes(dname, B_mean, P_mean, D_mean, NB_mean, geom.n_pix)
    peak, peak_kind = peaks()
    launch_s = dms / 1e3 / dcnt
    achieved = bytes_launch / launch_s / 1e9 if bytes_launch else None
    traffic, traffic_src = committed_traffic(dname, name, args.batch_cap)
    roofline = {
        "bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "peak_source": peak_kind,
        "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
        "traffic": traffic, "traffic_source": traffic_src,
        "traffic_ratio": (traffic / bytes_launch) if traffic and bytes_launch else None,
        "bytes_per_launch": bytes_launch, "mean_launch_us": launch_s * 1e6, "launches_per_step": dcnt,
        "share_of_serialised_step": dms / tot_ms if tot_ms else None,
        "batch_stats": {"events": B_mean, "evictions": P_mean, "distinct_pixels": D_mean, "blurs": NB_mean},
        "timing": "serialised engine (FIBAR_SERIAL=1, FIBAR_PDL=0), CUDA events around each launch",
    }
    R = 9 * geom.n_pix / (packet if per_packet else n)
    b_model = (21 + 24 * u_packet + 8 * blurs / n + R) if params.spatial_enabled else (13 + 16 * u_packet + R)
    path_achieved = value * 1e6 / world * b_model / 1e9
    path_roofline = {"bytes_per_event": b_model, "u_packet": u_packet, "blurs_per_event": blurs / n,
                     "achieved": path_achieved, "frac": path_achieved / peak, "unit": "GB/s",
                     "model": "SURVEY 8(d) B_ON = 21 + 24u + 8b + R / B_OFF = 13 + 16u + R"}

    e2e = None
    if not args.no_e2e:
        t_h = timed(step_host, max(1, args.steps), max(1, min(args.warmup, 2)))
        e2e = {"value": n * world * max(1, args.steps) / t_h / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(5 * n),
               "d2h_bytes_per_step": int((geom.n_pix + 16) * nfr),
               "ms_per_step": t_h / max(1, args.steps) * 1e3,
               "path": "pipeline.run() frame loop, host packets (pinned numpy views)" if per_packet
               else "process_array per host packet + render"}
        assert frame_hash(last_frame["f"].pixels) == gpu_hashes[-1], "device and host arms disagree"

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32+int64", "data": "synthetic (seeded stream, workloads.py; the paper's recordings are not public)",
        "config": {"workload": name, "events_per_step": n, "packet": packet, "device_batch_cap": args.batch_cap,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "flushed (256 MiB write) between timed steps",
                   "inputs": "HBM-resident packets, one allocation per packet"},
        "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline, "path_roofline": path_roofline,
        "clocks": clk.summary(),
        "kernel_ms_per_step_serialised": {k: round(v[0], 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])},
        "window": {"batches": b_batches, **{k: st1[k] for k in ("window_chunks", "window_reruns", "warm_pops", "coop_iters",
                                       "fix_rounds", "pops")}},
        "blur_count": blurs, "event_count": n,
    }
    check = {"gpu_frame_hashes": gpu_hashes, "gpu_digest": gpu_digest}
    return result, (geom, params, ev, packet), check


def cpu_reference(geom, params, ev, packet, steps=1, per_packet=False, frame_cb=None):
    """Time the C oracle (single-threaded restatement of the reference kernels)
    with the same read-out cadence as our arm.  frame_cb(k, pixels) runs outside
    the timed total.  Returns (times, engine of the last step)."""
    from oracle import oracle as orc
    n = len(ev)
    times = []
    eng = None
    for _ in range(steps):
        eng = orc.OracleEngine(geom.width, geom.height, params)
        excl = 0.0
        t0 = time.perf_counter()
        k = 0
        for a in range(0, n, packet):
            b = min(n, a + packet)
            eng.process_array(ev.t[a:b], ev.x[a:b], ev.y[a:b], ev.p[a:b])
            if per_packet:
                px, _, _ = eng.render("robust")
                if frame_cb:
                    c0 = time.perf_counter()
                    frame_cb(k, px)
                    excl += time.perf_counter() - c0
                k += 1
        if not per_packet:
            px, _, _ = eng.render("robust")
            if frame_cb:
                c0 = time.perf_counter()
                frame_cb(0, px)
                excl += time.perf_counter() - c0
        times.append(time.perf_counter() - t0 - excl)
    return times, eng


def filter_off_line(args, dev, dist, config, events=None, packet=None, readout=None):
    """A filter-OFF row of the metric: device-resident Mev/s of the config's
    stream with the spatial filter off, and the final state checked against the
    oracle (bit-exact)."""
    import torch
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    geom, params, ev, packet, name = workload(args, 0, config=config, events=events, packet=packet, spatial=False,
                                              readout=readout)
    n = len(ev)
    cuts = list(range(0, n, packet)) + [n]
    pk = separate_device_packets(ev, cuts, dev)
    eng = ReconstructionEngine(geom, params)
    stream = torch.cuda.current_stream(dev)
    frame = torch.empty((geom.height, geom.width), dtype=torch.uint8, device=dev)
    meta = torch.empty(4, dtype=torch.float64, device=dev)
    per_packet = readout == "packet"

    def step():
        eng.reset()
        af = None
        for blk in pk:
            eng.process_array(blk)
            if per_packet:
                af = eng.render_async("robust", out=frame, meta=meta)
        if per_packet:
            stream.wait_event(af.event)
        else:
            eng.render_device("robust", out=frame)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    t = device_timer(dev, stream, dist, flush)(step, args.steps, args.warmup)
    step()
    torch.cuda.synchronize()
    gpu = state_digest(eng.state_arrays())
    last = frame.cpu().numpy()
    eng.close()
    _, ref = cpu_reference(geom, params, ev, packet, per_packet=False)
    px, _, _ = ref.render("robust")
    ok = gpu == ref.state_digest() and frame_hash(last) == frame_hash(px)
    if not ok:
        raise SystemExit(f"filter-OFF parity mismatch on {name}")
    return {"workload": name, "value": n * args.steps / t / 1e6, "unit": UNIT,
            "ms_per_step": t / args.steps * 1e3, "parity": "exact (final state + last frame vs oracle)"}


def host_info() -> dict:
    """CPU model and host core count for the CPU-baseline lines."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "host_cores": os.cpu_count()}


def pinned_one_core():
    """Pin this process to one core for the single-threaded CPU baseline (as the
    survey's taskset -c recipe); returns the previous affinity to restore."""
    try:
        prev = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {min(prev)})
        return prev
    except (AttributeError, OSError):
        return None


def run_bands(args, rank, world, dist):
    """Filter OFF on N GPUs: row bands.  Every rank holds the whole
    packet stream (same seed) and its native engine keeps its own rows; the
    read-out all-gathers the bands over NCCL and renders the full frame."""
    import torch
    from paper_2510_20071_b200.bands import BandedReconstructionEngine
    from paper_2510_20071_b200.core import EventArray
    from paper_2510_20071_b200.pipeline import DeviceEventArray, render_grid

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    geom, params, ev, packet, name = workload(args, 0)
    n = len(ev)
    xd = torch.from_numpy(ev.x.view(np.int16)).to(dev)
    yd = torch.from_numpy(ev.y.view(np.int16)).to(dev)
    pd = torch.from_numpy(ev.p).to(dev)
    beng = BandedReconstructionEngine(geom, params, rank=rank, world=world, batch_capacity=args.batch_cap)
    eng = beng.engine
    stream = torch.cuda.current_stream(dev)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    cuts = list(range(0, n, packet)) + [n]
    xh = torch.from_numpy(ev.x.view(np.int16)).pin_memory().numpy().view(np.uint16)
    yh = torch.from_numpy(ev.y.view(np.int16)).pin_memory().numpy().view(np.uint16)
    ph = torch.from_numpy(ev.p).pin_memory().numpy()
    host_packets = [EventArray(ev.t[a:b], xh[a:b], yh[a:b], ph[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    frames = {}

    def step(host):
        eng.reset()
        if host:
            for blk in host_packets:
                beng.process_array(blk)
        else:
            for a, b in zip(cuts[:-1], cuts[1:]):
                beng.process_array(DeviceEventArray(xd[a:b], yd[a:b], pd[a:b]))
        full = beng.gather_l()
        if rank == 0:
            frames["f"] = render_grid(full, "robust")

    def timed(host, steps, warmup):
        for _ in range(warmup):
            step(host)
        torch.cuda.synchronize()
        total = 0.0
        for _ in range(steps):
            flush_buf.zero_()
            dist.barrier()
            torch.cuda.synchronize()
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step(host)
            s1.record(stream)
            torch.cuda.synchronize()
            total += s0.elapsed_time(s1) / 1e3
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    l0 = eng.stats()["launches"]
    with ClockSampler(dev.index) as clk:
        t_dev = timed(False, args.steps, args.warmup)
    launches = (eng.stats()["launches"] - l0) // (args.steps + args.warmup)
    t_h = timed(True, max(1, args.steps), 1)
    value = n * args.steps / t_dev / 1e6
    peak, peak_kind = peaks()
    R = 9 * geom.n_pix / n
    pid = ev.y.astype(np.int64) * geom.width + ev.x
    u_packet = float(np.mean([np.unique(pid[a:a + packet]).size / min(packet, n - a) for a in range(0, min(n, 50 * packet), packet)]))
    b_off = 13 + 16 * u_packet + R
    achieved = value * 1e6 * b_off / 1e9
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_dev / args.steps * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32+int64", "data": "synthetic (seeded stream, workloads.py)",
        "config": {"workload": name, "events_per_step": n, "packet": packet, "parallelism": f"row bands x{world}",
                   "l2": "flushed (256 MiB write) between timed steps",
                   "inputs": "every rank holds the whole packet stream in its HBM; each keeps its band's rows"},
        "e2e": {"value": n * max(1, args.steps) / t_h / 1e6, "unit": UNIT, "h2d_bytes_per_step": int(5 * n),
                "d2h_bytes_per_step": int(geom.n_pix + 16)},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "whole step (B_OFF model)", "achieved": achieved, "peak": peak,
                     "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak / world, "traffic": None},
        "clocks": clk.summary(),
    }


def run_halo_bands(args, rank, world, dist):
    """Filter ON on N GPUs: halo row bands.  Every rank holds the
    whole packet stream and runs the window pass on it; the blur is split by
    rows, the halo rows' blurred values go to the neighbours over NCCL in
    rounds until final, and the read-out all-gathers the bands."""
    import torch
    from paper_2510_20071_b200.bands import HaloBandEngine
    from paper_2510_20071_b200.core import EventArray
    from paper_2510_20071_b200.pipeline import DeviceEventArray, render_grid

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    geom, params, ev, packet, name = workload(args, 0)
    n = len(ev)
    xd = torch.from_numpy(ev.x.view(np.int16)).to(dev)
    yd = torch.from_numpy(ev.y.view(np.int16)).to(dev)
    pd = torch.from_numpy(ev.p).to(dev)
    beng = HaloBandEngine(geom, params, rank=rank, world=world, halo=args.halo, batch_events=args.halo_batch)
    eng = beng.engine
    stream = torch.cuda.current_stream(dev)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    B = beng.batch_events
    cuts = list(range(0, n, B)) + [n]
    xh = torch.from_numpy(ev.x.view(np.int16)).pin_memory().numpy().view(np.uint16)
    yh = torch.from_numpy(ev.y.view(np.int16)).pin_memory().numpy().view(np.uint16)
    ph = torch.from_numpy(ev.p).pin_memory().numpy()
    pcuts = list(range(0, n, packet)) + [n]
    host_packets = [EventArray(ev.t[a:b], xh[a:b], yh[a:b], ph[a:b]) for a, b in zip(pcuts[:-1], pcuts[1:])]
    frames = {}

    def step(host):
        eng.reset()
        beng.rounds.clear()
        if host:
            for blk in host_packets:
                beng.process_array(blk)
        else:
            # packets resident in HBM, handed over one device batch at a time
            for a, b in zip(cuts[:-1], cuts[1:]):
                beng.rounds.append(beng._run_batch(DeviceEventArray(xd[a:b], yd[a:b], pd[a:b])))
        full = beng.gather_l()
        if rank == 0:
            frames["f"] = render_grid(full, "robust")

    def timed(host, steps, warmup):
        for _ in range(warmup):
            step(host)
        torch.cuda.synchronize()
        total = 0.0
        for _ in range(steps):
            flush_buf.zero_()
            dist.barrier()
            torch.cuda.synchronize()
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step(host)
            s1.record(stream)
            torch.cuda.synchronize()
            total += s0.elapsed_time(s1) / 1e3
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    l0 = eng.stats()["launches"]
    with ClockSampler(dev.index) as clk:
        t_dev = timed(False, args.steps, args.warmup)
    launches = (eng.stats()["launches"] - l0) // (args.steps + args.warmup)
    rounds = list(beng.rounds)
    t_h = timed(True, max(1, args.steps), 1)
    value = n * args.steps / t_dev / 1e6
    peak, peak_kind = peaks()
    qs = eng.qs
    R = 9 * geom.n_pix / n
    pid = ev.y.astype(np.int64) * geom.width + ev.x
    u_packet = float(np.mean([np.unique(pid[a:a + packet]).size / min(packet, n - a) for a in range(0, min(n, 50 * packet), packet)]))
    b_on = 21 + 24 * u_packet + 8 * float(qs[5]) / n + R
    achieved = value * 1e6 * b_on / 1e9
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_dev / args.steps * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32+int64", "data": "synthetic (seeded stream, workloads.py)",
        "config": {"workload": name, "events_per_step": n, "packet": packet, "device_batch": B,
                   "parallelism": f"halo row bands x{world} (G={beng.halo})",
                   "l2": "flushed (256 MiB write) between timed steps",
                   "inputs": "every rank holds the whole packet stream in its HBM; window pass on every rank, "
                             "blur split by rows"},
        "e2e": {"value": n * max(1, args.steps) / t_h / 1e6, "unit": UNIT, "h2d_bytes_per_step": int(5 * n),
                "d2h_bytes_per_step": int(geom.n_pix + 16)},
        "gpu_launches": int(launches),
        "halo_rounds_per_batch": {"mean": float(np.mean(rounds)) if rounds else None,
                                  "max": int(max(rounds)) if rounds else None},
        "roofline": {"bound": "hbm", "kernel": "whole step (B_ON model)", "achieved": achieved, "peak": peak,
                     "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak / world, "traffic": None},
        "clocks": clk.summary(),
    }


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if args.impl == "reference":
        if rank != 0:
            return
        geom, params, ev, packet, name = workload(args, 0)
        prev = pinned_one_core()
        pp = args.readout == "packet"
        for _ in range(args.warmup):
            cpu_reference(geom, params, ev.slice(0, min(len(ev), 1_000_000)), packet, per_packet=pp)
        times, _ = cpu_reference(geom, params, ev, packet, steps=args.steps, per_packet=pp)
        if prev:
            os.sched_setaffinity(0, prev)
        v = len(ev) * args.steps / sum(times) / 1e6
        out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(times) / len(times) * 1e3,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+int64",
               "data": "synthetic (seeded stream, workloads.py; the paper's recordings are not public)",
               "config": {"workload": name, "events_per_step": len(ev), "packet": packet},
               "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"full workload ({len(ev)} events, same read-out cadence) x {args.steps} "
                                          "steps; C oracle (oracle/fibar_oracle.c) restating the reference's numba "
                                          "kernels and render, single thread pinned to one core like the "
                                          "single-threaded reference", **host_info()},
               "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return
    if world > 1 or args.bands:
        import torch.distributed as tdist
        if not tdist.is_initialized():
            if "MASTER_ADDR" not in os.environ:
                os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29511", RANK="0", WORLD_SIZE="1")
            tdist.init_process_group("nccl")
        dist = tdist
        cfg = workloads.CONFIGS[args.config]
        spatial = (args.filter == "on") if args.filter else (cfg["spatial"] if cfg["spatial"] is not None else True)
        if not args.replicas:
            line = (run_bands if not spatial else run_halo_bands)(args, rank, world, dist)
            if rank == 0:
                print(json.dumps(line))
            dist.destroy_process_group()
            return
    res = run_ours(args, rank, world, dist)
    if res is None:
        return
    result, (geom, params, ev, packet), check = res
    if rank == 0 and world == 1 and not args.no_cpu:
        per_packet = args.readout == "packet"
        cpu_hashes = []
        prev = pinned_one_core()
        times, ref = cpu_reference(geom, params, ev, packet, steps=1, per_packet=per_packet,
                                   frame_cb=lambda k, px: cpu_hashes.append(frame_hash(px)))
        if prev:
            os.sched_setaffinity(0, prev)
        v = len(ev) / times[0] / 1e6
        result["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                                  "sample": f"full workload ({len(ev)} events, one pass, same read-out cadence) "
                                            "pinned to one host core; C oracle restating the reference's numba "
                                            "kernels and render (frame hashing excluded from the time)",
                                  **host_info()}
        frames_ok = cpu_hashes == check["gpu_frame_hashes"]
        state_ok = ref.state_digest() == check["gpu_digest"]
        bad = [k for k, (a, b) in enumerate(zip(cpu_hashes, check["gpu_frame_hashes"])) if a != b]
        result["parity"] = {"state": "exact" if state_ok else "MISMATCH",
                            "frames": "exact" if frames_ok else f"MISMATCH at frames {bad[:5]}",
                            "n_frames": len(cpu_hashes), "events": len(ev),
                            "against": "C oracle (oracle/fibar_oracle.c) on the same stream and cadence; "
                                       "state = sha256 of p_bar, l, active_count, tile_count, qx, qy, qs"}
        if not (frames_ok and state_ok):
            print(json.dumps(result))
            raise SystemExit("parity mismatch between the CUDA path and the oracle")
    if rank == 0 and world == 1 and not args.no_off and args.config == 3 and args.events is None:
        import torch
        dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
        result["filter_off"] = {
            "config4_1M_packets": filter_off_line(args, dev, dist, 4, packet=1_000_000, readout="packet"),
            "config1": filter_off_line(args, dev, dist, 1),
        }
    if rank == 0:
        print(json.dumps(result))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
