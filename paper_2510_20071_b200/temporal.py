"""Per-pixel temporal filter utilities (reference `fibar/temporal.py`).

Same names, arguments and results as the reference module:

* ``PixelState``, ``update_pixel``, ``update_pixel_iir``,
  ``apply_threshold_map`` (temporal.py:25-67) are scalar float64 helpers --
  plain Python arithmetic in the same operation order, exactly as the
  reference defines them (there is nothing to put on a GPU in one scalar step).
* ``stream_pixel`` / ``stream_pixel_iir`` (temporal.py:78-117) run a polarity
  sequence through the recurrences on the device (``fibar_pixel_trace`` /
  ``fibar_pixel_trace_iir``, csrc/fibar_tools.cu) with the reference kernels'
  separately rounded operation order (_kernels.py:219-249), so float32 traces
  are bit-identical to the streaming engine and to the reference.
* ``stream_pixels`` / ``stream_pixels_iir`` take a (n_traces, n) polarity
  matrix and trace every row in parallel (one device thread per row).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import _native
from .core import FilterParams
from .errors import ConfigError, DataError


@dataclass(frozen=True)
class PixelState:
    """Filter memory of one pixel: detrend average, brightness, window membership."""

    p_bar: float = 0.0
    l: float = 0.0
    active_count: int = 0


def update_pixel(state: PixelState, polarity: int, params: FilterParams) -> tuple[PixelState, float]:
    """One event at one pixel (float64 scalars): returns (new state, detrended increment)."""
    if polarity not in (-1, 1):
        raise DataError(f"polarity must be -1 or +1, got {polarity}")
    p = float(polarity)
    new_p_bar = params.alpha * state.p_bar + (1.0 - params.alpha) * p
    delta = p - new_p_bar
    new_l = params.beta * state.l + params.half_one_plus_beta * delta
    return replace(state, p_bar=new_p_bar, l=new_l), delta


def update_pixel_iir(l_prev: float, l_prev2: float, polarity: int, polarity_prev: int,
                     params: FilterParams) -> float:
    """One step of the combined second-order recurrence (cross-check form)."""
    a, b = params.alpha, params.beta
    return (a + b) * l_prev - a * b * l_prev2 + 0.5 * a * (1.0 + b) * (polarity - polarity_prev)


def apply_threshold_map(delta: float, c_prime: float) -> float:
    """Scale a detrended increment by the pixel's relative threshold."""
    if not (c_prime > 0.0):
        raise DataError(f"relative threshold must be positive, got {c_prime}")
    return delta * c_prime


@dataclass
class PixelTrace:
    """Per-event trajectories of one pixel's filter state (2-D for batched traces)."""

    p_bar: np.ndarray
    delta: np.ndarray
    l: np.ndarray


def _dtype_code(dtype) -> tuple[np.dtype, int]:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return dt, 0
    if dt == np.float64:
        return dt, 1
    raise ConfigError(f"trace dtype must be float32 or float64, got {dt}")


def _torch_dtype(dt: np.dtype):
    import torch

    return torch.float32 if dt == np.float32 else torch.float64


def _polarity_matrix(polarities) -> np.ndarray:
    ps = np.asarray(polarities, dtype=np.int8)
    if ps.ndim == 1:
        ps = ps[None, :]
    if ps.ndim != 2:
        raise ConfigError("polarities must be a sequence or a (n_traces, n) matrix")
    return np.ascontiguousarray(ps)


def _device():
    import torch

    if not torch.cuda.is_available():
        from .errors import DeviceError
        raise DeviceError("pixel traces run on a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_pixels(polarities, params: FilterParams, dtype=np.float32) -> PixelTrace:
    """Trace every row of a (n_traces, n) polarity matrix from zero state."""
    import torch

    dt, code = _dtype_code(dtype)
    ps = _polarity_matrix(polarities)
    ntr, n = ps.shape
    dev = _device()
    tdt = _torch_dtype(dt)
    p_d = torch.from_numpy(ps).to(dev)
    state = torch.zeros((ntr, 2), dtype=tdt, device=dev)
    outs = [torch.empty((ntr, n), dtype=tdt, device=dev) for _ in range(3)]
    coef = (C.c_double * 4)(params.alpha, 1.0 - params.alpha, params.beta, params.half_one_plus_beta)
    lib = _native.load()
    stream = torch.cuda.current_stream(dev).cuda_stream
    _native.check(lib.fibar_pixel_trace(p_d.data_ptr(), n, ntr, code, coef, state.data_ptr(),
                                        outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(),
                                        C.c_void_p(stream)), "fibar_pixel_trace")
    pb, d, l = (o.cpu().numpy() for o in outs)
    return PixelTrace(pb, d, l)


def stream_pixel(polarities, params: FilterParams, dtype=np.float32) -> PixelTrace:
    """Run one polarity sequence through the two-stage filter from zero state.

    float32 matches the streaming engine bit for bit; float64 is the
    high-precision reference (temporal.py:78-100)."""
    tr = stream_pixels(np.asarray(polarities, dtype=np.int8).reshape(1, -1), params, dtype)
    return PixelTrace(tr.p_bar[0], tr.delta[0], tr.l[0])


def stream_pixels_iir(polarities, params: FilterParams, dtype=np.float32) -> np.ndarray:
    """Combined-recurrence traces of every row of a polarity matrix from zero state."""
    import torch

    dt, code = _dtype_code(dtype)
    ps = _polarity_matrix(polarities)
    ntr, n = ps.shape
    dev = _device()
    tdt = _torch_dtype(dt)
    p_d = torch.from_numpy(ps).to(dev)
    state = torch.zeros((ntr, 3), dtype=tdt, device=dev)
    out = torch.empty((ntr, n), dtype=tdt, device=dev)
    a, b = params.alpha, params.beta
    coef = (C.c_double * 3)(a + b, a * b, 0.5 * a * (1.0 + b))
    lib = _native.load()
    stream = torch.cuda.current_stream(dev).cuda_stream
    _native.check(lib.fibar_pixel_trace_iir(p_d.data_ptr(), n, ntr, code, coef, state.data_ptr(), out.data_ptr(),
                                            C.c_void_p(stream)), "fibar_pixel_trace_iir")
    return out.cpu().numpy()


def stream_pixel_iir(polarities, params: FilterParams, dtype=np.float32) -> np.ndarray:
    """Run one polarity sequence through the combined recurrence from zero state (temporal.py:103-117)."""
    return stream_pixels_iir(np.asarray(polarities, dtype=np.int8).reshape(1, -1), params, dtype)[0]
