"""Stereo depth from re-rendered baselines (stereo.py:1-219).

Same names, defaults and errors as the reference.  The second eye is the scene
re-rendered with the camera shifted along its own +x / +y axis; ZNCC block
matching (rcgs_stereo_match) recovers the disparity, which becomes depth and is
fused H/V by minimum (rcgs_stereo_depth).  Given the same images, disparities
are bit-identical to the reference's (the box means restate scipy's running-sum
uniform_filter, see csrc/stereo.cu).  `stereo_hv_depth` / `estimate_depth`
render the four images on the GPU (fp32 renders, so their disparities are those
of this renderer's images) and never leave the device until the result.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import device as D
from .errors import ValidationError
from .render import DEFAULT_CONFIG, DEFAULT_DEPTH_TAU, depth_from_gaussians, render
from .scene import CameraPose, scene_radius

INVALID_DISPARITY = -1.0


@dataclass(frozen=True)
class StereoConfig:
    """stereo.py:34-41."""

    baseline: float | None = None  # None: 2% of the scene bounding-sphere radius
    max_disparity: int = 64
    window_radius: int = 5
    variance_floor: float = 1e-6
    lr_tolerance: float = 1.0
    min_disparity: float = 1e-3


DEFAULT_STEREO = StereoConfig()


@dataclass(frozen=True)
class StereoPair:
    """A rectified pair; fx is the focal length along the baseline axis (stereo.py:47-54)."""

    left: np.ndarray
    right: np.ndarray
    baseline: float
    fx: float


def default_baseline(scene) -> float:
    return 0.02 * scene_radius(scene)


def _second_eye(intrinsics, pose, baseline: float, direction: str):
    """(shifted pose, focal along the baseline) -- stereo.py:64-78."""
    if baseline <= 0:
        raise ValidationError("baseline must be positive")
    axes = {"horizontal": (0, intrinsics.fx), "vertical": (1, intrinsics.fy)}
    if direction not in axes:
        raise ValidationError(f"unknown stereo direction {direction!r}")
    axis, focal = axes[direction]
    shift = np.zeros(3)
    shift[axis] = baseline
    return CameraPose(pose.rotation, np.asarray(pose.translation, np.float64) - shift), focal


def render_stereo_pair(scene, intrinsics, pose, baseline: float, direction: str = "horizontal",
                       config=DEFAULT_CONFIG) -> StereoPair:
    """The view and a second eye shifted by `baseline` in view space (stereo.py:61-84)."""
    right_pose, focal = _second_eye(intrinsics, pose, baseline, direction)
    return StereoPair(left=render(scene, intrinsics, pose, config=config),
                      right=render(scene, intrinsics, right_pose, config=config), baseline=baseline, fx=focal)


def _as_image(image) -> np.ndarray:
    a = np.asarray(image, dtype=np.float64)
    if a.ndim not in (2, 3):
        raise ValidationError(f"expected (H, W) or (H, W, 3) image, got {a.shape}")
    return np.ascontiguousarray(a)


def _match_device(left: torch.Tensor, right: torch.Tensor, height: int, width: int, ch_l: int, ch_r: int,
                  transpose: bool, config: StereoConfig, out=None) -> torch.Tensor:
    disp = out if out is not None else torch.empty((height, width), dtype=torch.float64, device=D.device())
    N.call("rcgs_stereo_match", N.ptr(left), N.ptr(right), height, width, ch_l, ch_r, left.element_size(),
           int(transpose), int(config.max_disparity), int(config.window_radius), float(config.variance_floor),
           float(config.variance_floor ** 2), float(config.lr_tolerance), N.ptr(disp), D.stream_ptr())
    return disp


def match_disparity(left, right, config: StereoConfig = DEFAULT_STEREO) -> np.ndarray:
    """ZNCC block matching; (H, W) float64 disparity, -1 where invalid (stereo.py:142-161)."""
    a, b = _as_image(left), _as_image(right)
    if a.shape[:2] != b.shape[:2]:
        raise ValidationError(f"stereo pair shapes differ: {a.shape[:2]} vs {b.shape[:2]}")
    h, w = a.shape[:2]
    ch_l, ch_r = (1 if x.ndim == 2 else x.shape[2] for x in (a, b))
    if h == 0 or w == 0 or ch_l == 0 or ch_r == 0:
        raise ValidationError(f"empty stereo image {a.shape}")
    dev = D.device()
    return _match_device(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev), h, w, ch_l, ch_r, False,
                         config).cpu().numpy()


def disparity_to_depth(disparity, fx: float, baseline: float,
                       min_disparity: float = DEFAULT_STEREO.min_disparity) -> np.ndarray:
    """depth = fx * baseline / disparity; invalid or tiny disparities give +inf (stereo.py:164-171)."""
    disparity = np.asarray(disparity, dtype=np.float64)
    depth = np.full(disparity.shape, np.inf)
    keep = disparity > min_disparity
    depth[keep] = fx * baseline / disparity[keep]
    return depth


def aggregate_hv(depth_h, depth_v) -> np.ndarray:
    """Pointwise minimum of the two estimates (stereo.py:174-181)."""
    depth_h = np.asarray(depth_h, dtype=np.float64)
    depth_v = np.asarray(depth_v, dtype=np.float64)
    if depth_h.shape != depth_v.shape:
        raise ValidationError(f"depth shapes differ: {depth_h.shape} vs {depth_v.shape}")
    return np.minimum(depth_h, depth_v)


def stereo_hv_depth_device(dscene, sh_dev, intrinsics, pose, baseline: float, config: StereoConfig = DEFAULT_STEREO,
                           raster=DEFAULT_CONFIG, backfill_tau: float | None = None) -> torch.Tensor:
    """(H, W) float64 device depth: H/V stereo fused by minimum; with backfill_tau,
    holes take the gaussian depth at that tau (estimate_depth "stereo-hv")."""
    h, w = int(intrinsics.height), int(intrinsics.width)
    dev = D.device()

    def image(p):
        v = D.View(dscene, intrinsics, p, raster)
        try:
            return v.color(sh_dev).render(None, 0)
        finally:
            v.close()

    pose_h, _ = _second_eye(intrinsics, pose, baseline, "horizontal")
    pose_v, _ = _second_eye(intrinsics, pose, baseline, "vertical")
    left = image(pose)
    disp_h = _match_device(left, image(pose_h), h, w, 3, 3, False, config)
    disp_v = _match_device(left, image(pose_v), h, w, 3, 3, True, config)
    fallback = None
    if backfill_tau is not None:
        v = D.View(dscene, intrinsics, pose, raster)
        try:
            fallback = v.depth(backfill_tau)
        finally:
            v.close()
    out = torch.empty((h, w), dtype=torch.float64, device=dev)
    N.call("rcgs_stereo_depth", N.ptr(disp_h), N.ptr(disp_v), h * w, float(intrinsics.fx * baseline),
           float(intrinsics.fy * baseline), float(config.min_disparity), N.ptr(fallback), N.ptr(out), D.stream_ptr())
    return out


def stereo_hv_depth(scene, intrinsics, pose, config: StereoConfig = DEFAULT_STEREO, raster=DEFAULT_CONFIG) -> np.ndarray:
    """Fused horizontal + vertical stereo depth, holes left as +inf (stereo.py:184-201)."""
    baseline = config.baseline if config.baseline is not None else default_baseline(scene)
    return stereo_hv_depth_device(D.device_scene(scene), D.sh_to_device(scene.sh), intrinsics, pose, baseline,
                                  config, raster).cpu().numpy()


def estimate_depth(scene, intrinsics, pose, method: str = "stereo-hv", tau: float = DEFAULT_DEPTH_TAU,
                   config: StereoConfig = DEFAULT_STEREO, raster=DEFAULT_CONFIG) -> np.ndarray:
    """"gaussians" (transmittance heuristic) or "stereo-hv" (fused stereo, holes
    backfilled from the gaussian depth) -- stereo.py:204-219."""
    if method == "gaussians":
        return depth_from_gaussians(scene, intrinsics, pose, tau, raster)
    if method == "stereo-hv":
        baseline = config.baseline if config.baseline is not None else default_baseline(scene)
        return stereo_hv_depth_device(D.device_scene(scene), D.sh_to_device(scene.sh), intrinsics, pose, baseline,
                                      config, raster, backfill_tau=tau).cpu().numpy()
    raise ValidationError(f"unknown depth method {method!r}")
