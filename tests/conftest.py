"""Shared fixtures.  `-m gpu` tests need a CUDA device and the built library;
everything else runs on the CPU (oracle, golden vectors, host logic, ABI)."""

from __future__ import annotations

import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and librcgs.so")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def golden_scene(d):
    return SimpleNamespace(positions=d["positions"], rotations=d["rotations"], scales=d["scales"],
                           opacities=d["opacities"], sh=d["sh"], sh_degree=int(d["sh_degree"]))


def golden_camera(d, prefix):
    K = d[prefix + "K"]
    intr = SimpleNamespace(fx=float(K[0]), fy=float(K[1]), cx=float(K[2]), cy=float(K[3]),
                           width=int(K[4]), height=int(K[5]))
    pose = SimpleNamespace(rotation=d[prefix + "R"], translation=d[prefix + "t"])
    return intr, pose


@pytest.fixture(scope="session")
def two_blobs():
    return load_golden("two_blobs_32.npz")


@pytest.fixture(scope="session")
def orbit_room():
    return load_golden("orbit_room_96.npz")


@pytest.fixture(scope="session")
def scaled_small():
    return load_golden("scaled_small.npz")


def identity_camera(width=32, height=32, fx=None):
    """Camera at the origin looking down +z (reference tests/conftest.py:39-45)."""
    fx = float(fx if fx is not None else width)
    intr = SimpleNamespace(fx=fx, fy=fx, cx=(width - 1) / 2.0, cy=(height - 1) / 2.0,
                           width=width, height=height)
    pose = SimpleNamespace(rotation=np.eye(3), translation=np.zeros(3))
    return intr, pose


def dc_sh(color):
    sh = np.zeros((16, 3))
    sh[0] = (np.asarray(color, dtype=np.float64) - 0.5) / 0.28209479177387814
    return sh


def make_scene(specs, sh_degree=3):
    """specs: list of dicts(position, color, scale, opacity, quat, sh)."""
    pos, rot, scl, opa, sh = [], [], [], [], []
    for s in specs:
        pos.append(np.asarray(s["position"], np.float64))
        rot.append(np.asarray(s.get("quat", (1.0, 0.0, 0.0, 0.0)), np.float64))
        sc = s.get("scale", 0.1)
        scl.append(np.full(3, sc) if np.isscalar(sc) else np.asarray(sc, np.float64))
        opa.append(float(s.get("opacity", 0.8)))
        sh.append(s["sh"] if "sh" in s else dc_sh(s.get("color", (1.0, 0.0, 0.0))))
    return SimpleNamespace(positions=np.array(pos).reshape(-1, 3), rotations=np.array(rot).reshape(-1, 4),
                           scales=np.array(scl).reshape(-1, 3), opacities=np.array(opa),
                           sh=np.array(sh).reshape(-1, 16, 3), sh_degree=sh_degree)


def pytest_sessionfinish(session, exitstatus):
    """Checked library builds (RCGS_LIB_PATH=.../checked/librcgs.so, compiled with
    -DRCGS_CHECKED): fail the run if any device bound check failed."""
    path = os.environ.get("RCGS_LIB_PATH", "")
    if "checked" not in path:
        return
    import ctypes
    lib = ctypes.CDLL(path)
    count = ctypes.c_uint64(0)
    rc = lib.rcgs_debug_violations(ctypes.byref(count), 1)
    # the counter itself: one deliberate failure must read back as 1
    lib.rcgs_debug_selftest(1)
    probe = ctypes.c_uint64(0)
    lib.rcgs_debug_violations(ctypes.byref(probe), 1)
    print(f"\nchecked build: rcgs_debug_violations rc={rc} count={count.value} (self-test reads {probe.value})")
    if rc != 0 or count.value != 0 or probe.value != 1:
        session.exitstatus = 1
