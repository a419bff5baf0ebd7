"""ctypes binding of ``librcgs.so`` (the C ABI declared in include/rcgs.h).

There is no CPU fallback: importing a compute entry point without the built
library, or without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading
import time

from .errors import SplattintError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
# RCGS_LIB_PATH: an alternate in-tree build for A/B measurements (tools/); the
# default is the library __graft_entry__.build() makes
LIB_PATH = os.environ.get("RCGS_LIB_PATH") or os.path.join(_HERE, "_lib", "librcgs.so")

RCGS_OK, RCGS_EINVAL, RCGS_ECUDA, RCGS_ENOMEM = 0, 1, 2, 3

c_void_p = ctypes.c_void_p
c_int = ctypes.c_int
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_double = ctypes.c_double
P = ctypes.POINTER


class Camera(ctypes.Structure):
    _fields_ = [("fx", c_double), ("fy", c_double), ("cx", c_double), ("cy", c_double),
                ("width", c_i32), ("height", c_i32), ("R", c_double * 9), ("t", c_double * 3)]


class RasterConfig(ctypes.Structure):
    _fields_ = [("near_clip", c_double), ("alpha_clamp", c_double), ("alpha_skip", c_double),
                ("transmittance_floor", c_double), ("covariance_dilation", c_double),
                ("footprint_sigmas", c_double)]


class AdamConfig(ctypes.Structure):
    _fields_ = [("lr_dc", c_double), ("lr_rest", c_double), ("beta1", c_double),
                ("beta2", c_double), ("eps", c_double)]


class AdamPublish(ctypes.Structure):
    _fields_ = [("d_snapshot", c_void_p), ("d_snapshot_step", c_void_p), ("every", c_i64)]


class ViewInfo(ctypes.Structure):
    _fields_ = [("n_gaussians", c_i64), ("n_kept", c_i64), ("n_pairs", c_i64),
                ("tiles_x", c_i32), ("tiles_y", c_i32), ("tile_size", c_i32), ("sort_bits", c_i32)]


# name -> (argtypes); every function returns int status except the two noted.
_SIGNATURES = {
    "rcgs_scene_create": [c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_int, c_void_p,
                          P(c_void_p)],
    "rcgs_scene_destroy": [c_void_p, c_void_p],
    "rcgs_view_create": [c_void_p, P(Camera), P(RasterConfig), c_void_p, P(c_void_p)],
    "rcgs_view_info_get": [c_void_p, P(ViewInfo)],
    "rcgs_view_destroy": [c_void_p, c_void_p],
    "rcgs_view_kept": [c_void_p, c_void_p, c_void_p, c_void_p],
    "rcgs_view_ranges": [c_void_p, c_void_p, c_void_p],
    "rcgs_view_pairs": [c_void_p, c_void_p, c_void_p],
    "rcgs_view_exact": [c_void_p, c_void_p, c_void_p],
    "rcgs_view_color": [c_void_p, c_void_p, c_void_p],
    "rcgs_render": [c_void_p, P(ctypes.c_float), c_int, c_void_p, c_void_p, c_void_p],
    "rcgs_view_keep_records": [c_void_p, c_void_p],
    "rcgs_render_rgba": [c_void_p, c_void_p, P(c_double), c_double, c_void_p, c_void_p],
    "rcgs_render_train": [c_void_p, P(ctypes.c_float), c_int, c_void_p, c_void_p, c_void_p],
    "rcgs_depth": [c_void_p, c_double, c_void_p, c_void_p, c_void_p],
    "rcgs_capture": [c_void_p, P(c_i64), c_void_p, c_void_p, c_void_p, c_void_p],
    "rcgs_loss_grad": [c_void_p, c_void_p, c_i32, c_i32, c_double, c_void_p, c_void_p, c_void_p],
    "rcgs_loss_grad_f64": [c_void_p, c_void_p, c_i32, c_i32, c_double, c_void_p, c_void_p, c_void_p],
    "rcgs_backward": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "rcgs_sh_grad": [c_void_p, c_void_p, P(c_double), c_void_p, c_void_p],
    "rcgs_adam_fused": [c_void_p, c_void_p, c_void_p, c_void_p, P(c_void_p), P(c_double), c_i32,
                        P(AdamConfig), c_void_p, c_void_p, c_void_p, c_void_p],
    "rcgs_adam_fused_next": [c_void_p, c_void_p, c_void_p, c_void_p, P(c_void_p), P(c_double), c_i32,
                             P(AdamConfig), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "rcgs_adam_fused_ex": [c_void_p, c_void_p, c_void_p, c_void_p, P(c_void_p), P(c_double), c_i32,
                           P(AdamConfig), c_void_p, c_void_p, c_void_p, c_void_p, P(AdamPublish), c_void_p,
                           c_void_p],
    "rcgs_adam_dense": [c_void_p, c_void_p, c_void_p, c_void_p, c_i64, P(AdamConfig), c_void_p,
                        c_void_p, c_void_p],
    "rcgs_nonfinite_check": [c_void_p, c_i64, c_void_p, c_void_p],
    "rcgs_ply_decode": [c_void_p, c_i64, c_i32, P(ctypes.c_int32), c_void_p, c_void_p, c_void_p,
                        P(c_i64), c_void_p],
    "rcgs_ply_encode_sh": [c_void_p, c_void_p, c_void_p, c_i64, c_i32, P(ctypes.c_int32), c_void_p, c_void_p],
    "rcgs_stereo_match": [c_void_p, c_void_p, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_double,
                          c_double, c_double, c_void_p, c_void_p],
    "rcgs_stereo_div_check": [c_i32, c_i64, ctypes.c_uint64, P(c_i64), c_void_p],
    "rcgs_stereo_depth": [c_void_p, c_void_p, c_i64, c_double, c_double, c_double, c_void_p, c_void_p, c_void_p],
    "rcgs_knn_mean_distances": [c_void_p, c_i64, c_i32, c_void_p, c_void_p],
    "rcgs_project_cloud": [c_void_p, c_i64, P(Camera), c_void_p, c_i32, c_double, c_void_p,
                           c_void_p],
    "rcgs_apply_recolor": [c_void_p, c_void_p, c_i64, P(ctypes.c_float), c_void_p, c_void_p],
    "rcgs_view_basis": [c_void_p, c_void_p, c_void_p, c_void_p],
    "rcgs_apply_recolor_f64": [c_void_p, c_void_p, c_i64, P(c_double), c_void_p, c_void_p],
    "rcgs_mask_hits": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "rcgs_raster_counters": [c_void_p],
    "rcgs_raster_trace": [c_void_p, c_i64],
    "rcgs_fp32_peak": [c_i32, P(c_double), c_void_p],
    "rcgs_pool_reserve": [c_i64, c_void_p],
    "rcgs_debug_violations": [P(ctypes.c_uint64), c_int],
    "rcgs_debug_selftest": [c_int],
}
EXPORTED = tuple(_SIGNATURES) + ("rcgs_version", "rcgs_last_error")

_lib = None
_lock = threading.Lock()


def load_library(require_gpu: bool = True):
    """Load librcgs.so (once).  Raises SplattintError when it is missing or,
    with `require_gpu`, when no CUDA device is visible."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise SplattintError(
                    f"CUDA library not built: {LIB_PATH} is missing (run __graft_entry__.build())")
            lib = ctypes.CDLL(LIB_PATH)
            for name, args in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = c_int
            lib.rcgs_version.restype = c_int
            lib.rcgs_version.argtypes = []
            lib.rcgs_last_error.restype = ctypes.c_char_p
            lib.rcgs_last_error.argtypes = []
            _lib = lib
    if require_gpu:
        import torch
        if not torch.cuda.is_available():
            raise SplattintError("paper_2511_18441_b200 needs a CUDA device (sm_100a); none is visible")
    return _lib


def check(status: int) -> None:
    if status == RCGS_OK:
        return
    msg = _lib.rcgs_last_error().decode(errors="replace")
    if status == RCGS_EINVAL:
        raise ValidationError(msg)
    raise SplattintError(f"rcgs error {status}: {msg}")


_CALL_TIMES = None  # {(thread name, fn): [max ms, count, total ms]} when profiling


def profile_calls(enable: bool = True) -> None:
    """Record host-side duration of every C-ABI call (diagnostics only)."""
    global _CALL_TIMES
    _CALL_TIMES = {} if enable else None


def call_times() -> dict:
    return dict(_CALL_TIMES or {})


def call(name: str, *args) -> None:
    lib = load_library()
    if _CALL_TIMES is None:
        check(getattr(lib, name)(*args))
        return
    t0 = time.perf_counter()
    rc = getattr(lib, name)(*args)
    ms = (time.perf_counter() - t0) * 1000.0
    key = (threading.current_thread().name, name)
    rec = _CALL_TIMES.setdefault(key, [0.0, 0, 0.0])
    rec[0] = max(rec[0], ms)
    rec[1] += 1
    rec[2] += ms
    check(rc)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()
