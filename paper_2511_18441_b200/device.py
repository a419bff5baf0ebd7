"""Device-side handles: scene geometry and per-view binned state.

PyTorch provides device memory and streams; every computation is a call into
librcgs.so (include/rcgs.h).  Geometry is frozen in the recolor workflow
(SH-only refit, optimize.py:1-12), so the device geometry is uploaded once per
distinct geometry (keyed on the identity of the host arrays, which
`Scene.with_sh` shares -- SURVEY.md 7.3.8) and every per-view structure
(projection, depth order, tile lists) is a `View` that can be reused across
SH updates: only `View.color` must be re-run after SH changes.
"""

from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict

import numpy as np
import torch

from . import _native as N
from .errors import ValidationError


def device() -> torch.device:
    N.load_library()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def camera_struct(intr, pose) -> N.Camera:
    cam = N.Camera()
    cam.fx, cam.fy, cam.cx, cam.cy = float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy)
    cam.width, cam.height = int(intr.width), int(intr.height)
    R = np.ascontiguousarray(pose.rotation, dtype=np.float64).ravel()
    t = np.ascontiguousarray(pose.translation, dtype=np.float64).ravel()
    for i in range(9):
        cam.R[i] = R[i]
    for i in range(3):
        cam.t[i] = t[i]
    return cam


def raster_struct(config) -> N.RasterConfig:
    c = N.RasterConfig()
    c.near_clip = config.near_clip
    c.alpha_clamp = config.alpha_clamp
    c.alpha_skip = config.alpha_skip
    c.transmittance_floor = config.transmittance_floor
    c.covariance_dilation = config.covariance_dilation
    c.footprint_sigmas = config.footprint_sigmas
    return c


def camera_center(pose) -> np.ndarray:
    """Same expression as CameraPose.camera_center (scene.py:72-75)."""
    return -np.asarray(pose.rotation, np.float64).T @ np.asarray(pose.translation, np.float64)


def to_device(arr, dtype=torch.float32) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(arr)).to(device=device(), dtype=dtype).contiguous()


class DeviceScene:
    """rcgs_scene: fp64 positions / opacities and the derived 3D covariances."""

    def __init__(self, positions, rotations, scales, opacities, sh_degree: int):
        dev = device()
        pos = torch.as_tensor(np.ascontiguousarray(positions, np.float64)).to(dev)
        rot = torch.as_tensor(np.ascontiguousarray(rotations, np.float64)).to(dev)
        scl = torch.as_tensor(np.ascontiguousarray(scales, np.float64)).to(dev)
        opa = torch.as_tensor(np.ascontiguousarray(opacities, np.float64)).to(dev)
        self.n = int(pos.shape[0])
        self.sh_degree = int(sh_degree)
        self.positions = pos  # kept for host-side helpers (directions, sharding)
        h = ctypes.c_void_p()
        N.call("rcgs_scene_create", N.ptr(pos), N.ptr(rot), N.ptr(scl), N.ptr(opa), self.n,
               self.sh_degree, stream_ptr(), ctypes.byref(h))
        self.handle = h
        torch.cuda.current_stream().synchronize()  # inputs may be freed after this

    @classmethod
    def from_device(cls, pos, rot, scl, opa, sh_degree: int) -> "DeviceScene":
        """From fp64 device tensors (N,3) positions, (N,4) unit rotations, (N,3) scales, (N,)."""
        self = cls.__new__(cls)
        self.n = int(pos.shape[0])
        self.sh_degree = int(sh_degree)
        self.positions = pos.contiguous()
        # the decoded geometry stays readable (checkpoint parity, host snapshots)
        self.rotations, self.scales, self.opacities = rot.contiguous(), scl.contiguous(), opa.contiguous()
        h = ctypes.c_void_p()
        N.call("rcgs_scene_create", N.ptr(self.positions), N.ptr(self.rotations), N.ptr(self.scales),
               N.ptr(self.opacities), self.n, self.sh_degree, stream_ptr(), ctypes.byref(h))
        self.handle = h
        torch.cuda.current_stream().synchronize()  # inputs may be freed after this
        return self

    @classmethod
    def from_scene(cls, scene) -> "DeviceScene":
        return cls(scene.positions, scene.rotations, scene.scales, scene.opacities, scene.sh_degree)

    def close(self):
        if getattr(self, "handle", None) and self.handle.value:
            N.load_library(require_gpu=False).rcgs_scene_destroy(self.handle, stream_ptr())
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_cache_lock = threading.Lock()
_scene_cache: "OrderedDict[tuple, tuple]" = OrderedDict()
_CACHE_SIZE = 4


def device_scene(scene) -> DeviceScene:
    """Cached DeviceScene for a host scene (keyed on geometry array identity)."""
    key = (id(scene.positions), id(scene.rotations), id(scene.scales), id(scene.opacities),
           int(scene.sh_degree), torch.cuda.current_device())
    with _cache_lock:
        hit = _scene_cache.get(key)
        if hit is not None:
            _scene_cache.move_to_end(key)
            return hit[1]
    ds = DeviceScene.from_scene(scene)
    with _cache_lock:
        # hold the host arrays so their ids cannot be recycled while cached
        _scene_cache[key] = ((scene.positions, scene.rotations, scene.scales, scene.opacities), ds)
        while len(_scene_cache) > _CACHE_SIZE:
            _scene_cache.popitem(last=False)
    return ds


def sh_to_device(sh) -> torch.Tensor:
    sh = torch.as_tensor(np.ascontiguousarray(sh)) if not isinstance(sh, torch.Tensor) else sh
    return sh.to(device=device(), dtype=torch.float32).contiguous()


class View:
    """One camera's preprocessed + binned gaussians (rcgs_view)."""

    def __init__(self, dscene: DeviceScene, intr, pose, config):
        self.scene = dscene
        self.intr = intr
        self.pose = pose
        self.width, self.height = int(intr.width), int(intr.height)
        self.center = camera_center(pose)
        h = ctypes.c_void_p()
        cam = camera_struct(intr, pose)
        cfg = raster_struct(config)
        N.call("rcgs_view_create", dscene.handle, ctypes.byref(cam), ctypes.byref(cfg), stream_ptr(),
               ctypes.byref(h))
        self.handle = h
        info = N.ViewInfo()
        N.call("rcgs_view_info_get", h, ctypes.byref(info))
        self.n_kept = int(info.n_kept)
        self.n_pairs = int(info.n_pairs)
        self.sort_bits = int(info.sort_bits)
        self.tiles = (int(info.tiles_x), int(info.tiles_y))
        self._colored = False

    # -- per SH state ----------------------------------------------------------
    def color(self, sh_dev: torch.Tensor) -> "View":
        if sh_dev.dtype != torch.float32 or not sh_dev.is_contiguous():
            raise ValidationError("device SH must be contiguous float32 (N, 16, 3)")
        N.call("rcgs_view_color", self.handle, N.ptr(sh_dev), stream_ptr())
        self._colored = True
        return self

    def _need_color(self):
        if not self._colored:
            raise ValidationError("View.color(sh) must run before rendering")

    # -- raster ----------------------------------------------------------------
    def render(self, background=None, layout: int = 0, out=None, t_final=False, train: bool = False):
        """Composite the view.  train=True also keeps its composite weights
        (rcgs_render_train) so backward() streams them instead of re-traversing."""
        self._need_color()
        shape = (self.height, self.width, 3) if layout == 0 else (3, self.height, self.width)
        img = out if out is not None else torch.empty(shape, dtype=torch.float32, device=device())
        tf = torch.empty((self.height, self.width), dtype=torch.float32, device=device()) if t_final else None
        bg = (ctypes.c_float * 3)(*(np.zeros(3) if background is None else np.asarray(background, np.float64)))
        N.call("rcgs_render_train" if train else "rcgs_render", self.handle, bg, int(layout), N.ptr(img),
               N.ptr(tf), stream_ptr())
        return (img, tf) if t_final else img

    def render_rgba(self, overlay=None, highlight=(1.0, 0.8, 0.1), strength: float = 0.45, out=None):
        """Viewer frame (session.py:381-405 render_rgba): the view composited on a
        zero background, `overlay` (H,W) pixels blended toward `highlight`, then
        quantised to (H,W,4) uint8 RGBA (protocol.py image_to_rgba) -- one pass
        (rcgs_render_rgba)."""
        self._need_color()
        rgba = out if out is not None else torch.empty((self.height, self.width, 4), dtype=torch.uint8,
                                                         device=device())
        ov = None
        if overlay is not None:
            ov = overlay if overlay.dtype == torch.uint8 else overlay.to(torch.uint8)
            ov = ov.contiguous()
        hl = (ctypes.c_double * 3)(*[float(c) for c in highlight])
        N.call("rcgs_render_rgba", self.handle, N.ptr(ov), hl, float(strength), N.ptr(rgba), stream_ptr())
        return rgba

    def keep_records(self):
        """Keep the composite weights recorded by a train render resident with the
        view (rcgs_view_keep_records): later renders / backwards stream them."""
        if not getattr(self, "_records_kept", False):
            N.call("rcgs_view_keep_records", self.handle, stream_ptr())
            self._records_kept = True

    def depth(self, tau: float = 0.5, with_cross: bool = False):
        d = torch.empty((self.height, self.width), dtype=torch.float64, device=device())
        c = torch.empty((self.height, self.width), dtype=torch.int32, device=device()) if with_cross else None
        N.call("rcgs_depth", self.handle, float(tau), N.ptr(d), N.ptr(c), stream_ptr())
        return (d, c) if with_cross else d

    def capture(self):
        """Contribution lists (pixel, kept rank, weight) as device tensors."""
        count = ctypes.c_int64(0)
        N.call("rcgs_capture", self.handle, ctypes.byref(count), None, None, None, stream_ptr())
        n = count.value
        dev = device()
        pix = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        kept = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        w = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        count = ctypes.c_int64(n)
        N.call("rcgs_capture", self.handle, ctypes.byref(count), N.ptr(pix), N.ptr(kept), N.ptr(w),
               stream_ptr())
        return pix[:n], kept[:n], w[:n]

    def kept(self):
        idx = torch.empty(max(self.n_kept, 1), dtype=torch.int64, device=device())
        z = torch.empty(max(self.n_kept, 1), dtype=torch.float64, device=device())
        N.call("rcgs_view_kept", self.handle, N.ptr(idx), N.ptr(z), stream_ptr())
        return idx[:self.n_kept], z[:self.n_kept]

    def ranges(self) -> torch.Tensor:
        """Per-tile [start, end) into the depth-ordered pair list, (tiles_y, tiles_x, 2)."""
        out = torch.zeros((self.tiles[1], self.tiles[0], 2), dtype=torch.int32, device=device())
        if self.n_pairs:
            N.call("rcgs_view_ranges", self.handle, N.ptr(out), stream_ptr())
        return out

    def pairs(self) -> torch.Tensor:
        """The binned pair list: scene indices sorted by (tile, depth rank)."""
        out = torch.zeros(max(self.n_pairs, 1), dtype=torch.int32, device=device())
        if self.n_pairs:
            N.call("rcgs_view_pairs", self.handle, N.ptr(out), stream_ptr())
        return out[:self.n_pairs]

    def exact(self) -> torch.Tensor:
        """(K, 6) fp64 mean2d x, y, conic a, b, c, opacity of the kept gaussians in depth order."""
        out = torch.zeros((max(self.n_kept, 1), 6), dtype=torch.float64, device=device())
        if self.n_kept:
            N.call("rcgs_view_exact", self.handle, N.ptr(out), stream_ptr())
        return out[:self.n_kept]

    def backward(self, grad_image: torch.Tensor, acc=None, nonfinite=None) -> torch.Tensor:
        self._need_color()
        if tuple(grad_image.shape) != (self.height, self.width, 3):
            raise ValidationError(
                f"gradient image shape {tuple(grad_image.shape)} does not match render "
                f"{(self.height, self.width, 3)}")
        g = grad_image.to(dtype=torch.float32).contiguous()
        acc = acc if acc is not None else torch.empty((self.scene.n, 3), dtype=torch.float32, device=device())
        N.call("rcgs_backward", self.handle, N.ptr(g), N.ptr(acc), N.ptr(nonfinite), stream_ptr())
        return acc

    def mask_hits(self, mask_u8: torch.Tensor, hits: torch.Tensor, wsum: torch.Tensor):
        N.call("rcgs_mask_hits", self.handle, N.ptr(mask_u8), N.ptr(hits), N.ptr(wsum), stream_ptr())

    def close(self):
        if getattr(self, "handle", None) and self.handle.value:
            N.load_library(require_gpu=False).rcgs_view_destroy(self.handle, stream_ptr())
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def loss_grad(image: torch.Tensor, target: torch.Tensor, lam: float, loss3=None, grad=None):
    """rcgs_loss_grad on device HWC float32 tensors -> (loss3 fp64 device, grad fp32)."""
    h, w = int(image.shape[0]), int(image.shape[1])
    dev = image.device
    loss3 = loss3 if loss3 is not None else torch.empty(3, dtype=torch.float64, device=dev)
    grad = grad if grad is not None else torch.empty_like(image)
    N.call("rcgs_loss_grad", N.ptr(image), N.ptr(target), h, w, float(lam), N.ptr(loss3), N.ptr(grad),
           stream_ptr())
    return loss3, grad


def adam_config(config) -> N.AdamConfig:
    c = N.AdamConfig()
    c.lr_dc, c.lr_rest = config.lr_dc, config.lr_rest
    c.beta1, c.beta2, c.eps = config.beta1, config.beta2, config.eps
    return c
