"""Selection pass + edited datasets (drop-in for splattint/recolor.py).

Per view (recolor.py:59-81): K4 depth (exact fp64 crossing z) -> K8 cloud
projection with occlusion test (bit-exact mask) -> recolour of the masked
ground truth.  `SelectionPass` is the device-resident engine used by the
optimizer and the benchmark: views keep their binned state (geometry is
frozen), targets stay in HBM as float32, and the per-gaussian mask statistics
(hit counts, integer-exact; masked contribution weight, 2^-32 fixed point) are
accumulated across views -- sharded across ranks they reduce exactly with one
integer all-reduce.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import device as D
from .errors import ValidationError
from .render import DEFAULT_CONFIG, DEFAULT_DEPTH_TAU
from .selection import DEFAULT_DEPTH_TOLERANCE, DEFAULT_QUAD_SIZE, project_cloud_device


def _check_tint(tint) -> np.ndarray:
    tint = np.asarray(tint, dtype=np.float64)
    if tint.shape != (3,):
        raise ValidationError(f"tint must be 3 components, got shape {tint.shape}")
    if not np.all(np.isfinite(tint)) or np.any(tint < 0):
        raise ValidationError("tint components must be finite and >= 0")
    return tint


def apply_recolor_device(image: torch.Tensor, mask_u8: torch.Tensor, tint, out=None) -> torch.Tensor:
    """out = mask ? clip(image * tint, 0, 1) : image on device (fp32 or fp64 HWC)."""
    tint = _check_tint(tint)
    out = out if out is not None else torch.empty_like(image)
    npix = int(image.shape[0]) * int(image.shape[1])
    if image.dtype == torch.float64:
        N.call("rcgs_apply_recolor_f64", N.ptr(image), N.ptr(mask_u8), npix, (ctypes.c_double * 3)(*tint),
               N.ptr(out), D.stream_ptr())
    else:
        N.call("rcgs_apply_recolor", N.ptr(image), N.ptr(mask_u8), npix, (ctypes.c_float * 3)(*tint),
               N.ptr(out), D.stream_ptr())
    return out


def apply_recolor(image, mask, tint) -> np.ndarray:
    """recolor.py:30-39 (fp64, bit-exact)."""
    tint = _check_tint(tint)
    image = np.asarray(image, dtype=np.float64)
    mask = np.asarray(mask, dtype=bool)
    if mask.shape != image.shape[:2]:
        raise ValidationError(f"mask shape {mask.shape} does not match image {image.shape[:2]}")
    if image.ndim != 3 or image.shape[2] != 3:
        raise ValidationError(f"expected (H, W, 3) image, got {image.shape}")
    out = apply_recolor_device(D.to_device(image, torch.float64), D.to_device(mask, torch.uint8), tint)
    return out.cpu().numpy()


@dataclass(frozen=True)
class EditedView:
    view: object        # TrainingView
    mask: np.ndarray    # (H, W) bool
    image: np.ndarray   # (H, W, 3) recoloured ground truth


@dataclass(frozen=True)
class EditedDataset:
    views: tuple
    generation: int
    tint: np.ndarray

    def __len__(self) -> int:
        return len(self.views)


def build_edited_dataset(views, cloud, tint, scene, generation: int = 0,
                         quad_size: int = DEFAULT_QUAD_SIZE,
                         depth_tolerance: float = DEFAULT_DEPTH_TOLERANCE,
                         tau: float = DEFAULT_DEPTH_TAU, raster=DEFAULT_CONFIG) -> EditedDataset:
    """Project the cloud into every view and recolour the masked pixels (recolor.py:59-81)."""
    tint = _check_tint(tint)
    edited = []
    pts = None if cloud.is_empty else D.to_device(cloud.points, torch.float64)
    ds = None if cloud.is_empty else D.device_scene(scene)
    for view in views:
        h, w = view.intrinsics.height, view.intrinsics.width
        img = D.to_device(view.image, torch.float64)
        if pts is None:
            mask = torch.zeros((h, w), dtype=torch.uint8, device=img.device)
        else:
            dv = D.View(ds, view.intrinsics, view.pose, raster)
            depth = dv.depth(tau)
            mask = project_cloud_device(pts, view.intrinsics, view.pose, depth, quad_size,
                                        depth_tolerance)
        out = apply_recolor_device(img, mask, tint)
        edited.append(EditedView(view=view, mask=mask.cpu().numpy().astype(bool), image=out.cpu().numpy()))
    return EditedDataset(views=tuple(edited), generation=generation, tint=tint)


class SelectionPass:
    """Device-resident selection pass over a set of cameras.

    Holds one `device.View` per camera (reused by the optimizer), the float32
    ground truth (V, H, W, 3), and after `run`: masks (V, H, W) uint8, the
    edited targets (V, H, W, 3) float32 and optional per-gaussian statistics.
    """

    def __init__(self, dscene: D.DeviceScene, cameras, gt: torch.Tensor, raster=DEFAULT_CONFIG,
                 views=None, keep_views: bool = False):
        self.dscene = dscene
        self.cameras = list(cameras)
        self.gt = gt
        self.raster = raster
        self.keep_views = keep_views or views is not None
        self.views = views if views is not None else [None] * len(self.cameras)
        self.masks = None
        self.edited = None
        self.hits = None
        self.wsum = None

    def view(self, i: int) -> D.View:
        if self.views[i] is None:
            intr, pose = self.cameras[i]
            self.views[i] = D.View(self.dscene, intr, pose, self.raster)
        return self.views[i]

    def run(self, points_dev: torch.Tensor, tint, indices=None, quad_size: int = DEFAULT_QUAD_SIZE,
            depth_tolerance: float = DEFAULT_DEPTH_TOLERANCE, tau: float = DEFAULT_DEPTH_TAU,
            stats: bool = True):
        """Selection over `indices` (default all views)."""
        tint = _check_tint(tint)
        dev = D.device()
        idx = range(len(self.cameras)) if indices is None else indices
        v, h, w = self.gt.shape[0], self.gt.shape[1], self.gt.shape[2]
        if self.masks is None:
            self.masks = torch.zeros((v, h, w), dtype=torch.uint8, device=dev)
            self.edited = self.gt.clone()
        if stats and self.hits is None:
            self.hits = torch.zeros(self.dscene.n, dtype=torch.int32, device=dev)
            self.wsum = torch.zeros(self.dscene.n, dtype=torch.int64, device=dev)
        idx = list(idx)
        has_points = points_dev is not None and points_dev.shape[0] > 0
        # views not kept are built ahead on side streams by worker threads (their
        # two host syncs and latency-bound build kernels overlap this loop's
        # depth / projection / hit passes); results are identical
        pf = None
        ahead = 3
        if has_points and not self.keep_views and len(idx) > 1 and all(self.views[i] is None for i in idx):
            from .engine import ViewPrefetcher  # engine imports this module's users, not this module
            # the views in flight come from the retained pool (as RefitEngine reserves)
            N.call("rcgs_pool_reserve", int((ahead + 2) * self.dscene.n * 400), D.stream_ptr())
            pf = ViewPrefetcher(self.dscene, self.cameras, self.raster, dev.index if dev.index is not None else 0,
                                depth=ahead)
            for k, i in enumerate(idx[:ahead]):
                pf.submit(k, i)
        try:
            for k, i in enumerate(idx):
                intr, pose = self.cameras[i]
                self.masks[i].zero_()
                if has_points:
                    if pf is not None:
                        view, ev, _ = pf.take(k)
                        torch.cuda.current_stream().wait_event(ev)
                        if k + ahead < len(idx):
                            pf.submit(k + ahead, idx[k + ahead])
                    else:
                        view = self.view(i)
                    depth = view.depth(tau)
                    project_cloud_device(points_dev, intr, pose, depth, quad_size, depth_tolerance,
                                         out=self.masks[i])
                    if stats:
                        view.mask_hits(self.masks[i], self.hits, self.wsum)
                    if pf is not None:
                        pf.retire(view)
                    elif not self.keep_views:
                        view.close()
                        self.views[i] = None
                apply_recolor_device(self.gt[i], self.masks[i], tint, out=self.edited[i])
        finally:
            if pf is not None:
                pf.close()
        return self

    def wsum_float(self) -> torch.Tensor:
        return self.wsum.double() / 4294967296.0
