"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/rcgs.h declares; host-side API validation behaves like the
reference; host helpers agree with the oracle.  No kernel launches."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
import paper_2511_18441_b200 as P
from paper_2511_18441_b200 import _native
from oracle import raster as OR, selection as OS


def header_symbols():
    text = open(os.path.join(ROOT, "include", "rcgs.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(rcgs_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _native.load_library(require_gpu=False)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _native.EXPORTED, f"{s} not bound in _native"
    assert lib.rcgs_version() == 1


def test_library_is_sm100a_only():
    so = _native.LIB_PATH
    out = os.popen(f"cuobjdump --list-elf {so} 2>&1").read()
    assert "sm_100a" in out, out


def test_compute_entry_points_fail_loudly_without_gpu(monkeypatch):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.SplattintError, match="CUDA device"):
        _native.load_library(require_gpu=True)


def test_scene_validation_matches_reference():
    ok = dict(positions=np.zeros((1, 3)), rotations=np.array([[1.0, 0, 0, 0]]), scales=np.ones((1, 3)),
              opacities=np.array([0.5]), sh=np.zeros((1, 16, 3)))
    P.Scene(**ok)
    for field, bad in [("opacities", np.array([1.0])), ("scales", np.zeros((1, 3))),
                       ("rotations", np.array([[2.0, 0, 0, 0]])), ("sh", np.zeros((1, 15, 3))),
                       ("positions", np.full((1, 3), np.nan))]:
        with pytest.raises(P.ValidationError):
            P.Scene(**{**ok, field: bad})
    with pytest.raises(P.ValidationError):
        P.CameraIntrinsics(10, 10, 20, 5, 16, 16)
    with pytest.raises(P.ValidationError):
        P.CameraPose(np.diag([1.0, 1.0, -1.0]), np.zeros(3))


def test_host_helpers_match_oracle():
    rng = np.random.default_rng(0)
    d = rng.normal(size=(50, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    for deg in range(4):
        np.testing.assert_array_equal(P.sh_basis(d, deg), OR.sh_basis(d, deg))
    q = rng.normal(size=(20, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    np.testing.assert_array_equal(P.quaternion_to_rotation(q), OR.quat_to_rot(q))
    img = rng.normal(size=(5, 7, 3))
    np.testing.assert_array_equal(P.from_chw(P.to_chw(img)), img)
    with pytest.raises(P.ValidationError):
        P.to_chw(np.zeros((3, 4, 4)))


def test_select_from_mask_host_steps_match_oracle(two_blobs):
    from conftest import golden_camera
    intr, pose = golden_camera(two_blobs, "v0_")
    depth = two_blobs["v0_depth"]
    intr_p = P.CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)
    pose_p = P.CameraPose(pose.rotation, pose.translation)
    mask = P.SelectionMask2D(two_blobs["brush"], intr_p, pose_p)
    # unproject is host numpy (the seeded permutation is numpy's); the outlier
    # filter's kNN runs on the GPU (tests/test_gpu_parity.py)
    cloud = P.unproject(mask, depth, 0.7, 0)
    np.testing.assert_array_equal(cloud.points, OS.unproject(two_blobs["brush"], depth, intr, pose, 0.7, 0))
    tiny = P.SelectionCloud(cloud.points[:10])
    with pytest.warns(UserWarning):  # <= k points: returned unchanged, no GPU needed
        assert P.remove_outliers(tiny, 16, 1.0) is tiny
    with pytest.raises(P.ValidationError):
        P.remove_outliers(cloud, 0, 1.0)
    disc = P.apply_stroke(P.new_mask(intr_p, pose_p), "brush", [(10.0, 12.0)], 4.0).bits
    np.testing.assert_array_equal(disc, OS.stroke_disc(intr.height, intr.width, (10.0, 12.0), 4.0))


def test_metrics_line_format():
    m = P.IterationMetrics(iteration=3, view_id=1, generation=0,
                           loss=P.LossBreakdown(l1=0.1, ssim=0.9, total=0.1, lam=0.2))
    assert re.fullmatch(r"\d+,\d+,\d+,\d+\.\d{8},-?\d+\.\d{8},\d+\.\d{8}", m.line())
