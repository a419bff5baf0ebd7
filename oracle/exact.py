"""ctypes wrappers of the C restatement of the exact-decision arithmetic
(oracle/c/rcgs_oracle.c) -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

`project_exact` returns, per gaussian, every fp64 value the reference's
preprocess feeds into a discrete decision (render.py:172-214): z, mean2d,
dilated cov2d, det, the 3-sigma viewport test and the conic.  The tests pin it
bitwise to numpy / the reference (tests/test_oracle_golden.py) and the device
preprocess bitwise to it (tests/test_gpu_scale.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .config import COV_DILATION, FOOTPRINT_SIGMAS, NEAR_CLIP

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

FIELDS = ("kept", "z", "mx", "my", "a", "b", "c", "det", "ca", "cb", "cc", "radius")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "c", "librcgs_oracle.so")
        if not os.path.exists(path):
            subprocess.check_call(["make"], cwd=os.path.dirname(path))
        _LIB = ctypes.CDLL(path)
        d, i64, i32, vp = ctypes.c_double, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        _LIB.rcgs_oracle_cov3d.argtypes = [vp, vp, i64, vp]
        _LIB.rcgs_oracle_project_exact.argtypes = [vp, vp, i64, vp, vp, d, d, d, d, i32, i32, d, d, d, vp]
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def cov3d(rotations, scales) -> np.ndarray:
    """(N, 6) xx xy xz yy yz zz, bit-identical to render.py:95-100."""
    rot = np.ascontiguousarray(rotations, np.float64)
    scl = np.ascontiguousarray(scales, np.float64)
    out = np.empty((len(rot), 6))
    lib().rcgs_oracle_cov3d(_p(rot), _p(scl), len(rot), _p(out))
    return out


def project_exact(scene, intr, pose) -> dict:
    """Per-gaussian exact preprocess values (dict of (N,) arrays, FIELDS)."""
    pos = np.ascontiguousarray(scene.positions, np.float64)
    c3 = cov3d(scene.rotations, scene.scales)
    R = np.ascontiguousarray(pose.rotation, np.float64)
    t = np.ascontiguousarray(pose.translation, np.float64)
    out = np.empty((len(pos), 12))
    lib().rcgs_oracle_project_exact(_p(pos), _p(c3), len(pos), _p(R), _p(t), float(intr.fx), float(intr.fy),
                                    float(intr.cx), float(intr.cy), int(intr.width), int(intr.height),
                                    NEAR_CLIP, COV_DILATION, FOOTPRINT_SIGMAS, _p(out))
    res = {f: out[:, i] for i, f in enumerate(FIELDS)}
    res["kept"] = res["kept"].astype(bool)
    return res
