"""Rendering API (drop-in for splattint/render.py) on the sm_100a kernels.

`render`, `render_forward` and `depth_from_gaussians` keep the reference
signatures (render.py:304-398) and return float64 numpy arrays; internally
they build one `device.View` (K1 preprocess + K2 tile binning) and run the K3/K4
rasteriser.  The small per-gaussian helpers (`sh_basis`, `eval_sh`,
`compute_covariance`, `project_gaussian`, layout conversions) are host-side
conveniences of the reference API and are not on the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from .errors import ValidationError
from .scene import quaternion_to_rotation

SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
         -1.0925484305920792, 0.5462742152960396)
SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
         0.3731763325901154, -0.4570457994644658, 1.445305721320277, -0.5900435899266435)


@dataclass(frozen=True)
class RasterizerConfig:
    """render.py:54-66."""

    near_clip: float = 0.2
    alpha_clamp: float = 0.99
    alpha_skip: float = 1.0 / 255.0
    transmittance_floor: float = 1e-4
    covariance_dilation: float = 0.3
    footprint_sigmas: float = 3.0


DEFAULT_CONFIG = RasterizerConfig()
DEFAULT_DEPTH_TAU = 0.5


@dataclass(frozen=True)
class ProjectedGaussian:
    mean2d: np.ndarray
    conic: np.ndarray
    depth: float
    color: np.ndarray
    base_alpha: float


class ForwardCapture:
    """render_forward result (render.py:81-92).

    `image` is materialised eagerly; the per-contribution lists, basis and
    activation flags stay on the device and are copied to numpy only when an
    attribute is read.  `backward_sh` consumes the device state directly.
    """

    def __init__(self, view: D.View, image: np.ndarray, n_gaussians: int):
        self._view = view
        self.image = image
        self.n_gaussians = n_gaussians
        self._lists = None
        self._kept = None
        self._basis = None

    def _load_lists(self):
        if self._lists is None:
            pix, kept, w = self._view.capture()
            self._lists = (pix.cpu().numpy(), kept.cpu().numpy(), w.cpu().numpy())
        return self._lists

    def _load_basis(self):
        if self._basis is None:
            k = self._view.n_kept
            basis = torch.empty((max(k, 1), 16), dtype=torch.float64, device=D.device())
            active = torch.empty((max(k, 1), 3), dtype=torch.uint8, device=D.device())
            from . import _native as N
            N.call("rcgs_view_basis", self._view.handle, N.ptr(basis), N.ptr(active), D.stream_ptr())
            self._basis = (basis[:k].cpu().numpy(), active[:k].cpu().numpy().astype(bool))
        return self._basis

    @property
    def kept_index(self) -> np.ndarray:
        if self._kept is None:
            self._kept = self._view.kept()[0].cpu().numpy()
        return self._kept

    @property
    def basis(self) -> np.ndarray:
        return self._load_basis()[0]

    @property
    def active(self) -> np.ndarray:
        return self._load_basis()[1]

    @property
    def contrib_pixel(self) -> np.ndarray:
        return self._load_lists()[0]

    @property
    def contrib_kept(self) -> np.ndarray:
        return self._load_lists()[1]

    @property
    def contrib_weight(self) -> np.ndarray:
        return self._load_lists()[2]


def _background(background) -> np.ndarray:
    if background is None:
        return np.zeros(3)
    bg = np.asarray(background, dtype=np.float64)
    if bg.shape != (3,):
        raise ValidationError(f"background must be 3 floats, got shape {bg.shape}")
    return bg


def make_view(scene, intrinsics, pose, config=DEFAULT_CONFIG, sh=None) -> D.View:
    """Device view of a host scene; colours it from `sh` (default scene.sh)."""
    view = D.View(D.device_scene(scene), intrinsics, pose, config)
    view.color(D.sh_to_device(scene.sh if sh is None else sh))
    return view


def _host_image(view: D.View, bg: np.ndarray) -> np.ndarray:
    """HWC float64: the composite plus T_final * background added in float64, so a
    pixel no gaussian reaches equals the background bit-for-bit (render.py:317-322)."""
    if not np.any(bg):
        return view.render(None, 0).double().cpu().numpy()
    img, tf = view.render(None, 0, t_final=True)
    return img.double().cpu().numpy() + tf.double().cpu().numpy()[..., None] * bg


def render(scene, intrinsics, pose, background=None, config: RasterizerConfig = DEFAULT_CONFIG,
           layout: str = "hwc") -> np.ndarray:
    """(H, W, 3) float64, or (3, H, W) for layout="chw" (render.py:304-334)."""
    if layout not in ("hwc", "chw"):
        raise ValidationError(f"unknown layout {layout!r}")
    bg = _background(background)
    img = _host_image(make_view(scene, intrinsics, pose, config), bg)
    return img if layout == "hwc" else to_chw(img)


def render_forward(scene, intrinsics, pose, background=None,
                   config: RasterizerConfig = DEFAULT_CONFIG) -> ForwardCapture:
    """Render + device-resident contribution state (render.py:337-370)."""
    bg = _background(background)
    view = make_view(scene, intrinsics, pose, config)
    return ForwardCapture(view, _host_image(view, bg), len(scene))


def depth_from_gaussians(scene, intrinsics, pose, tau: float = DEFAULT_DEPTH_TAU,
                         config: RasterizerConfig = DEFAULT_CONFIG) -> np.ndarray:
    """(H, W) float64 depth of the first composited gaussian with T < tau, +inf
    elsewhere (render.py:373-398).  Exact: the returned values are the
    reference's fp64 view-space z of the crossing gaussian."""
    view = D.View(D.device_scene(scene), intrinsics, pose, config)
    return view.depth(tau).cpu().numpy()


# ---- host-side helpers of the reference API (not on the hot path) ---------------

def compute_covariance(rotation, scale) -> np.ndarray:
    """R S S^T R^T (render.py:95-100)."""
    m = quaternion_to_rotation(rotation) * np.asarray(scale, np.float64)[..., None, :]
    return m @ np.swapaxes(m, -1, -2)


def sh_basis(directions, degree: int) -> np.ndarray:
    """Real SH basis (..., 16), zero beyond `degree` (render.py:103-137)."""
    if not (0 <= degree <= 3):
        raise ValidationError("sh degree must be in [0, 3]")
    d = np.asarray(directions, dtype=np.float64)
    out = np.zeros(d.shape[:-1] + (16,))
    out[..., 0] = SH_C0
    if degree == 0:
        return out
    x, y, z = d[..., 0], d[..., 1], d[..., 2]
    out[..., 1:4] = np.stack([-SH_C1 * y, SH_C1 * z, -SH_C1 * x], -1)
    if degree == 1:
        return out
    xx, yy, zz, xy, yz, xz = x * x, y * y, z * z, x * y, y * z, x * z
    out[..., 4:9] = np.stack([SH_C2[0] * xy, SH_C2[1] * yz, SH_C2[2] * (2.0 * zz - xx - yy),
                              SH_C2[3] * xz, SH_C2[4] * (xx - yy)], -1)
    if degree == 2:
        return out
    out[..., 9:16] = np.stack([
        SH_C3[0] * y * (3.0 * xx - yy), SH_C3[1] * xy * z, SH_C3[2] * y * (4.0 * zz - xx - yy),
        SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy), SH_C3[4] * x * (4.0 * zz - xx - yy),
        SH_C3[5] * z * (xx - yy), SH_C3[6] * x * (xx - 3.0 * yy)], -1)
    return out


def eval_sh(coeffs, direction, degree: int = 3) -> np.ndarray:
    return np.einsum("...k,...kc->...c", sh_basis(direction, degree), np.asarray(coeffs, np.float64))


def color_activation(raw) -> np.ndarray:
    return np.maximum(0.0, np.asarray(raw, dtype=np.float64) + 0.5)


def project_gaussian(gaussian, intrinsics, pose,
                     config: RasterizerConfig = DEFAULT_CONFIG) -> ProjectedGaussian | None:
    """Screen-space footprint of one gaussian or None when culled (render.py:232-254)."""
    R, t = pose.rotation, pose.translation
    p =(np.asarray(gaussian.position, np.float64)[None] @ R.T + t)[0]
    x, y, z = p
    if not z > config.near_clip:
        return None
    mean2d = np.array([intrinsics.fx * x / z + intrinsics.cx, intrinsics.fy * y / z + intrinsics.cy])
    cov3 = compute_covariance(gaussian.rotation, gaussian.scale)
    jac = np.array([[intrinsics.fx / z, 0.0, -intrinsics.fx * x / (z * z)],
                    [0.0, intrinsics.fy / z, -intrinsics.fy * y / (z * z)]])
    tj = jac @ R
    cov2 = tj @ cov3 @ tj.T + config.covariance_dilation * np.eye(2)
    a, b, c = cov2[0, 0], cov2[0, 1], cov2[1, 1]
    det = a * c - b * b
    mid = 0.5 * (a + c)
    radius = config.footprint_sigmas * np.sqrt(mid + np.sqrt(max(mid * mid - det, 0.0)))
    if not (det > 0 and mean2d[0] + radius >= 0 and mean2d[0] - radius <= intrinsics.width - 1
            and mean2d[1] + radius >= 0 and mean2d[1] - radius <= intrinsics.height - 1):
        return None
    d = np.asarray(gaussian.position, np.float64) - pose.camera_center
    d = d / np.linalg.norm(d)
    raw = sh_basis(d, 3) @ np.asarray(gaussian.sh, np.float64)
    return ProjectedGaussian(mean2d=mean2d, conic=np.array([[c, -b], [-b, a]]) / det,
                             depth=float(z), color=color_activation(raw),
                             base_alpha=float(gaussian.opacity))


def to_chw(image) -> np.ndarray:
    image = np.asarray(image)
    if image.ndim != 3 or image.shape[2] != 3:
        raise ValidationError(f"to_chw expects (H, W, 3), got {image.shape}")
    return np.ascontiguousarray(np.transpose(image, (2, 0, 1)))


def from_chw(planes) -> np.ndarray:
    planes = np.asarray(planes)
    if planes.ndim != 3 or planes.shape[0] != 3:
        raise ValidationError(f"from_chw expects (3, H, W), got {planes.shape}")
    return np.ascontiguousarray(np.transpose(planes, (1, 2, 0)))
