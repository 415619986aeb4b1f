"""ctypes binding of the C ABI in include/fibar_b200.h.

The shared library is built in-tree (``python -m paper_2510_20071_b200.build``
or ``__graft_entry__.build()``) at ``paper_2510_20071_b200/_lib/libfibar_b200.so``.
There is no CPU fallback: if the library or a CUDA device is missing, the first
engine construction raises :class:`~.errors.DeviceError`.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import DeviceError, raise_for_status

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libfibar_b200.so")

FIBAR_MEM_HOST = 0
FIBAR_MEM_DEVICE = 1
FIBAR_RENDER_ROBUST = 0
FIBAR_RENDER_FIXED = 1

EXPORTED = (
    "fibar_create", "fibar_destroy", "fibar_set_stream", "fibar_reset", "fibar_process", "fibar_flush",
    "fibar_render", "fibar_read_qs", "fibar_counters", "fibar_read_state", "fibar_stats",
    "fibar_brightness_ptr", "fibar_last_error", "fibar_profile", "fibar_profile_read", "fibar_pending", "fibar_debug_times", "fibar_debug_prep", "fibar_debug_readout_times", "fibar_render_grid", "fibar_copy_brightness", "fibar_decode_evf1",
    "fibar_count_events", "fibar_pixel_trace", "fibar_pixel_trace_iir",
    "fibar_halo_batch", "fibar_halo_round", "fibar_halo_finish", "fibar_render_async", "fibar_debug_stale_items", "fibar_debug_trace",
    "fibar_debug_regulate",
)


class FibarConfig(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("tile_side", C.c_int32),
        ("spatial_enabled", C.c_int32),
        ("blur_enabled", C.c_int32),
        ("reserved0", C.c_int32),
        ("regulate_every", C.c_int64),
        ("fill_num", C.c_int64),
        ("fill_den", C.c_int64),
        ("q_min", C.c_int64),
        ("q_max", C.c_int64),
        ("alpha", C.c_float),
        ("one_m_alpha", C.c_float),
        ("beta", C.c_float),
        ("half_1p_beta", C.c_float),
        ("gain", C.c_void_p),
        ("batch_capacity", C.c_int64),
        ("band_y0", C.c_int32),
        ("sensor_height", C.c_int32),
        ("halo_own_y0", C.c_int32),
        ("halo_own_y1", C.c_int32),
        ("halo_rows", C.c_int32),
        ("reserved1", C.c_int32),
    ]


# The engine runs a batch on about a dozen CUDA streams; with the driver's
# default of 8 hardware queues, streams that share a queue serialise falsely
# (measured: the two ingest streams ran back to back).  Only effective when set
# before the CUDA context is created; a C caller sets it in its own environment.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

_lib = None


def load(path: str | None = None):
    """Load (once) and type the native library; raises DeviceError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("FIBAR_LIB") or LIB_PATH   # FIBAR_LIB: an alternative build (experiments)
    if not os.path.exists(path):
        raise DeviceError(f"native library {path} not built; run __graft_entry__.build()")
    L = C.CDLL(path)
    P, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "fibar_create": ([C.POINTER(FibarConfig), P, C.POINTER(P)], C.c_int),
        "fibar_destroy": ([P], C.c_int),
        "fibar_set_stream": ([P, P], C.c_int),
        "fibar_reset": ([P], C.c_int),
        "fibar_process": ([P, P, P, P, i64, i32], C.c_int),
        "fibar_flush": ([P], C.c_int),
        "fibar_render": ([P, i32, f64, P, i32, P, P], C.c_int),
        "fibar_read_qs": ([P, P], C.c_int),
        "fibar_counters": ([P, P, P], C.c_int),
        "fibar_read_state": ([P, P, P, P, P, P, P], C.c_int),
        "fibar_stats": ([P, P], C.c_int),
        "fibar_brightness_ptr": ([P, C.POINTER(P)], C.c_int),
        "fibar_last_error": ([], C.c_char_p),
        "fibar_profile": ([P, i32], C.c_int),
        "fibar_pending": ([P, P, P], C.c_int),
        "fibar_debug_times": ([P, P, P, i64], C.c_int),
        "fibar_debug_prep": ([P, P, i64], C.c_int),
        "fibar_debug_readout_times": ([P, P], C.c_int),
        "fibar_render_grid": ([P, i64, i32, f64, P, i32, P, P, P], C.c_int),
        "fibar_copy_brightness": ([P, P, i32], C.c_int),
        "fibar_decode_evf1": ([P, i64, i32, i32, C.c_uint64, P, P, P, P, P, P], C.c_int),
        "fibar_profile_read": ([P, i32, P, i32, P, P, P], C.c_int),
        "fibar_count_events": ([P, P, P, i64, i32, i64, P, P, P, P], C.c_int),
        "fibar_pixel_trace": ([P, i64, i32, i32, P, P, P, P, P, P], C.c_int),
        "fibar_pixel_trace_iir": ([P, i64, i32, i32, P, P, P, P], C.c_int),
        "fibar_halo_batch": ([P, P, P, P, i64, i32, P], C.c_int),
        "fibar_halo_round": ([P, i32, P, P], C.c_int),
        "fibar_halo_finish": ([P], C.c_int),
        "fibar_render_async": ([P, i32, f64, P, i32, P, P], C.c_int),
        "fibar_debug_stale_items": ([P, P, P, i64, P], C.c_int),
        "fibar_debug_regulate": ([i64, i64, i32, i64, i64, P, P, P, i64, P, P], C.c_int),
        "fibar_debug_trace": ([P, i64, P, P, P, P], C.c_int),
    }
    for name, (args, res) in sig.items():
        if path != LIB_PATH and not hasattr(L, name):
            continue   # an older experimental build (FIBAR_LIB) without this entry point
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(code: int, what: str) -> None:
    if code:
        msg = load().fibar_last_error().decode(errors="replace")
        try:
            raise_for_status(code, what)
        except Exception as exc:  # attach the native message
            raise type(exc)(f"{exc}: {msg}") from None
