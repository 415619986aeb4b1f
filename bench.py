"""Benchmark of the FIBAR reconstruction hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

Workload (BASELINE.json configs[1], the config the metric is quoted on):
640x480 sensor, 10M events of the seeded moving-texture stream
(paper_2510_20071_b200/workloads.py), spatial filter ON, 10k-event packets,
robust read-out at the end of the stream.  One *step* = reset the engine,
push all 1,000 packets through ``ReconstructionEngine.process_array``, render.

* ``value``: packets already resident in HBM (DeviceEventArray), frame left on
  the device; per-step CUDA events on the engine stream, L2 flushed (256 MiB
  write) between steps, summed over K steps, max over ranks.
* ``e2e``: the same step through the public host API: packets as numpy views
  of pinned host memory (H2D inside the timed region), Frame copied back.
* ``roofline``: the dominant kernel by device time (per-kernel CUDA events in an
  extra, untimed profiled step) -- its essential bytes per launch / its mean
  launch time, against MEASURED_PEAKS.json hbm_gbs.  ``path_roofline`` applies
  SURVEY §8(d)'s per-event byte model to the whole step.
* ``cpu_baseline``: the C oracle (a restatement of the reference's numba
  kernels, single thread by design) on the same 10M-event workload.

``--impl reference`` times that CPU implementation alone (rank 0; other ranks
exit) and prints the same JSON shape with ``"impl": "reference"``.
Multi-GPU: filter OFF runs row bands (strong scaling).  Filter
ON runs N independent replicas by default (seeds rank, weak scaling): the
window is one global FIFO and both of the step's chains are latency-bound, so
``--bands`` (halo row bands, exact, NCCL halo exchange) is available but not
faster than one GPU.
"""

from __future__ import annotations

import argparse
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
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--events", type=int, default=None, help="override the config's event count")
    ap.add_argument("--packet", type=int, default=None)
    ap.add_argument("--filter", default=None, choices=("on", "off"))
    ap.add_argument("--batch-cap", type=int, default=0, help="device batch capacity (0: the engine's default)")
    ap.add_argument("--readout", default=None, choices=("end", "packet"),
                    help="robust read-out at the end of the stream or after every packet (config default)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="one step, for ncu launch lists")
    ap.add_argument("--bands", action="store_true",
                    help="row bands (filter OFF: the default at N>1; filter ON: halo bands instead of replicas)")
    ap.add_argument("--halo", type=int, default=16, help="halo rows of the filter-ON row bands")
    ap.add_argument("--halo-batch", type=int, default=1 << 20, help="events per halo-band batch")
    return ap.parse_args()


def workload(args, rank):
    cfg = workloads.CONFIGS[args.config]
    geom = cfg["geometry"]
    n = args.events or cfg["n"]
    spatial = cfg["spatial"] if cfg["spatial"] is not None else True
    if args.filter:
        spatial = args.filter == "on"
    packet = args.packet or cfg["packet"] or 100_000
    kw = {"speed": cfg["speed"]} if "speed" in cfg else {}
    ev = workloads.make(cfg["kind"], geom, n, seed=rank, **kw)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=spatial)
    args.readout = args.readout or cfg.get("readout", "end")
    ro = "robust read-out after every packet" if args.readout == "packet" else "robust read-out at end"
    name = f"config{args.config}:{geom.width}x{geom.height},{n // 1_000_000}M events,{cfg['kind']}," \
           f"filter {'on' if spatial else 'off'},{packet}-event packets,{ro}"
    return geom, params, ev, packet, name


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling via NVML during the timed region."""

    def __init__(self, index=0, period=0.05):
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
            time.sleep(self.period)

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


# essential bytes per launch of each kernel: the data it must read and write
# once, from the batch statistics (B events, P evictions, D distinct pixels)
def kernel_bytes(name, B, P, D, n_pix):
    table = {
        "count_inb": 4 * B,
        "compact": 5 * B + 4 * B * 3 + 4 * B,          # read x,y,p; write key, tkey, pol, ring key
        "rs_hist": 4 * B,
        "rs_scatter": 8 * B + 8 * B,
        "seg_marks": 8 * B + 8 * D,
        "link": 8 * B + 16 * D + 8 * B + 8 * B,         # sorted keys/idx, pixel records, dp, ring next
        "anchor": 8 * B,
        "window_run": 8 * B + 8 * P + 4 * B,            # dp, ring next of evictions, window starts
        "popj": 4 * B + 12 * P,
        "temporal": 8 * B + 5 * B + 16 * D,            # sorted idx/pol, t2/L0 writes, p_bar/l RMW
        "blur": P * (4 + 8 + 4 + 8) + 9 * 4 * P,      # eviction item, ring next/key, 3x3 taps of l
        "final": 8 * B + 24 * D,
        "sel_hist": 4 * n_pix,
        "render_map": 5 * n_pix,
    }
    return table.get(name)


def committed_traffic(kernel: str, batch_cap: int, config: int):
    """DRAM bytes per launch of `kernel` from the latest committed ncu --set full
    capture (profiles/rNN*_traffic.json, latest round tag, written by scripts/summarize_ncu.py from
    `bench.py --profile-only`: config 2 at the default device batch); None for any
    other workload or an explicit batch size, or when no capture is committed."""
    import glob
    import json
    if batch_cap or config != 2:   # an explicit --batch-cap: not the captured workload
        return None
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "*_traffic.json")))
    for f in reversed(files):
        try:
            v = json.load(open(f))["bytes_per_launch"].get(kernel)
        except (OSError, ValueError, KeyError):
            continue
        if v:
            return v
    return None


def run_ours(args, rank, world, dist):
    import torch
    from paper_2510_20071_b200.core import EventArray
    from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine, run

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    geom, params, ev, packet, name = workload(args, rank)
    n = len(ev)
    xd = torch.from_numpy(ev.x.view(np.int16)).to(dev)
    yd = torch.from_numpy(ev.y.view(np.int16)).to(dev)
    pd = torch.from_numpy(ev.p).to(dev)
    eng = ReconstructionEngine(geom, params, batch_capacity=args.batch_cap)
    cap_explicit = args.batch_cap
    args.batch_cap = eng._bcap   # the effective device batch capacity
    stream = torch.cuda.current_stream(dev)
    frame = torch.empty((geom.height, geom.width), dtype=torch.uint8, device=dev)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    cuts = list(range(0, n, packet)) + [n]
    # the step's packets, resident in HBM before timing (views of one buffer)
    dev_packets = [DeviceEventArray(xd[a:b], yd[a:b], pd[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]

    per_packet = args.readout == "packet"

    meta_dev = torch.empty(4, dtype=torch.float64, device=dev)

    def step_device():
        eng.reset()
        if per_packet:
            # a read-out after every packet, enqueued asynchronously behind the
            # packet's blur stage (the next packet's front end overlaps it);
            # the step ends when the last frame is in HBM
            af = None
            for blk in dev_packets:
                eng.process_array(blk)
                af = eng.render_async("robust", out=frame, meta=meta_dev)
            stream.wait_event(af.event)
            return
        for blk in dev_packets:
            eng.process_array(blk)
        eng.render_device("robust", out=frame)

    # host arm: pinned host columns, numpy views per packet
    xh = torch.from_numpy(ev.x.view(np.int16)).pin_memory().numpy().view(np.uint16)
    yh = torch.from_numpy(ev.y.view(np.int16)).pin_memory().numpy().view(np.uint16)
    ph = torch.from_numpy(ev.p).pin_memory().numpy()
    th = ev.t
    host_packets = [EventArray(th[a:b], xh[a:b], yh[a:b], ph[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    last_frame = {}

    # per-packet read-outs go through the reference's own frame loop, run()
    # (pipeline.run: frames at each packet's end time, delivered to the host)
    pp_times = [int(ev.t[b - 1]) + 1 for b in cuts[1:]]

    def step_host():
        eng.reset()
        if per_packet:
            run(eng, host_packets, readout_times=pp_times, frame_sink=lambda k, f: last_frame.__setitem__("f", f))
            return
        for blk in host_packets:
            eng.process_array(blk)
        last_frame["f"] = eng.render("robust")

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

    if args.profile_only:
        step_device()
        torch.cuda.synchronize()
        return None

    l0 = eng.stats()["launches"]
    with ClockSampler(dev.index) as clk:
        t_dev = timed(step_device, args.steps, args.warmup)
    launches = (eng.stats()["launches"] - l0) // (args.steps + args.warmup)
    st = eng.stats()
    value = n * world * args.steps / t_dev / 1e6
    ms_per_step = t_dev / args.steps * 1e3

    # batch statistics for the byte model (from one more device step)
    step_device()
    qs = eng.qs
    blur_per_ev = float(qs[5]) / n
    pops_per_ev = 1.0  # refined below from stats
    st2 = eng.stats()
    b_batches = max(1, st2["batches"] - st["batches"])
    pops_per_ev = (st2["pops"] - st["pops"]) / n if st2["pops"] > st["pops"] else pops_per_ev
    pid = ev.y.astype(np.int64) * geom.width + ev.x
    Bcap = args.batch_cap
    u = float(np.mean([np.unique(pid[a:a + Bcap]).size / min(Bcap, n - a) for a in range(0, n, Bcap)]))
    u_packet = float(np.mean([np.unique(pid[a:a + packet]).size / min(packet, n - a) for a in range(0, min(n, 50 * packet), packet)]))

    # per-kernel device time (untimed profiled step)
    eng.profile(True)
    step_device()
    prof = eng.profile_read()
    eng.profile(False)
    tot_ms = sum(v[0] for v in prof.values())
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dname, (dms, dcnt) = dom
    B_mean = n / b_batches
    P_mean = pops_per_ev * B_mean
    D_mean = u * B_mean
    bytes_launch = kernel_bytes(dname, B_mean, P_mean, D_mean, geom.n_pix)
    peak, peak_kind = peaks()
    launch_s = dms / 1e3 / dcnt
    achieved = bytes_launch / launch_s / 1e9 if bytes_launch else None
    roofline = {
        "bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "peak_source": peak_kind,
        "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
        "traffic": committed_traffic(dname, cap_explicit, args.config),
        "share_of_step": dms / tot_ms if tot_ms else None, "mean_launch_us": launch_s * 1e6,
        "bytes_per_launch": bytes_launch,
    }
    R = 9 * geom.n_pix / (packet if per_packet else n)
    b_on = 21 + 24 * u_packet + 8 * blur_per_ev + R if params.spatial_enabled else 13 + 16 * u_packet + R
    path_achieved = value * 1e6 / world * b_on / 1e9
    path_roofline = {"bytes_per_event": b_on, "u_packet": u_packet, "u_batch": u, "blurs_per_event": blur_per_ev,
                     "achieved": path_achieved, "frac": path_achieved / peak, "unit": "GB/s", "model": "SURVEY 8(d) B_ON/B_OFF"}

    e2e = None
    if not args.no_e2e:
        t_h = timed(step_host, max(1, args.steps), 1)
        e2e = {"value": n * world * max(1, args.steps) / t_h / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(5 * n),
               "d2h_bytes_per_step": int((geom.n_pix + 16) * (len(host_packets) if per_packet else 1)),
               "ms_per_step": t_h / max(1, args.steps) * 1e3}
        # the two arms must agree
        fd = frame.cpu().numpy()
        assert np.array_equal(fd, last_frame["f"].pixels), "device and host arms disagree"

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32+int64", "data": "synthetic (seeded moving-texture stream, workloads.py)",
        "config": {"workload": name, "events_per_step": n, "packet": packet, "device_batch_cap": args.batch_cap,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "flushed (256 MiB write) between timed steps", "inputs": "HBM-resident packets"},
        "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline, "path_roofline": path_roofline,
        "clocks": clk.summary(),
        "kernel_ms_per_step": {k: round(v[0], 4) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])},
        "window": {k: st2[k] for k in ("window_chunks", "window_reruns", "warm_pops", "coop_iters", "fix_rounds", "pops")},
        "blur_count": int(qs[5]), "event_count": n,
    }
    return result, (geom, params, ev, packet)


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


def cpu_reference(geom, params, ev, packet, steps=1, per_packet=False):
    """Time the C oracle (single-threaded restatement of the reference kernels),
    with the same read-out cadence as our arm."""
    from oracle import oracle as orc
    n = len(ev)
    times = []
    for _ in range(steps):
        eng = orc.OracleEngine(geom.width, geom.height, params)
        t0 = time.perf_counter()
        for a in range(0, n, packet):
            b = min(n, a + packet)
            eng.process_array(ev.t[a:b], ev.x[a:b], ev.y[a:b], ev.p[a:b])
            if per_packet:
                eng.render("robust")
        if not per_packet:
            eng.render("robust")
        times.append(time.perf_counter() - t0)
    return times


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
        times = cpu_reference(geom, params, ev, packet, steps=args.steps, per_packet=pp)
        if prev:
            os.sched_setaffinity(0, prev)
        v = len(ev) * args.steps / sum(times) / 1e6
        out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(times) / len(times) * 1e3,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+int64",
               "data": "synthetic (seeded moving-texture stream, workloads.py)",
               "config": {"workload": name, "events_per_step": len(ev), "packet": packet},
               "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"full workload ({len(ev)} events) x {args.steps} steps; C oracle "
                                          "(oracle/fibar_oracle.c), single thread pinned to one core, as the "
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
        if not spatial or args.bands:
            line = (run_bands if not spatial else run_halo_bands)(args, rank, world, dist)
            if rank == 0:
                print(json.dumps(line))
            dist.destroy_process_group()
            return
    res = run_ours(args, rank, world, dist)
    if res is None:
        return
    result, (geom, params, ev, packet) = res
    if rank == 0 and world == 1 and not args.no_cpu:
        prev = pinned_one_core()
        times = cpu_reference(geom, params, ev, packet, steps=1, per_packet=args.readout == "packet")
        if prev:
            os.sched_setaffinity(0, prev)
        v = len(ev) / times[0] / 1e6
        result["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                                  "sample": f"full workload ({len(ev)} events, one pass) pinned to one host "
                                            "core; C oracle restating the reference's numba kernels",
                                  **host_info()}
    if rank == 0:
        print(json.dumps(result))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
