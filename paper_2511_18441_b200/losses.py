"""Photometric loss API (drop-in for splattint/losses.py) on the K5 kernel.

total = (1 - lam) L1 + lam (1 - SSIM); the loss, the SSIM map and the image
gradient are one fp64 kernel chain (csrc/loss.cu).  Host images are
kept in float64 for this host-facing API (the optimizer's device path uses the
float32 variant on float32 renders).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from .errors import ValidationError

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2
DEFAULT_LAMBDA = 0.2


@dataclass(frozen=True)
class LossBreakdown:
    l1: float
    ssim: float
    total: float
    lam: float


def gaussian_window(size: int = SSIM_WINDOW, sigma: float = SSIM_SIGMA) -> np.ndarray:
    """losses.py:41-45."""
    off = np.arange(size, dtype=np.float64) - size // 2
    k = np.exp(-(off ** 2) / (2.0 * sigma ** 2))
    return k / k.sum()


def _pair(image, reference, window: bool):
    image = np.asarray(image, dtype=np.float64)
    reference = np.asarray(reference, dtype=np.float64)
    if image.shape != reference.shape:
        raise ValidationError(f"image shapes differ: {image.shape} vs {reference.shape}")
    if image.ndim != 3 or image.shape[2] != 3:
        raise ValidationError(f"expected (H, W, 3) images, got {image.shape}")
    if window and min(image.shape[0], image.shape[1]) < SSIM_WINDOW:
        raise ValidationError(f"images must be at least {SSIM_WINDOW}px on each side for SSIM")
    return D.to_device(image, torch.float64), D.to_device(reference, torch.float64)


def _lam(lam):
    if not (0.0 <= lam <= 1.0):
        raise ValidationError("lam must be in [0, 1]")


def _run(image, reference, lam, window):
    """float64 images in, float64 gradient out (rcgs_loss_grad_f64)."""
    from . import _native as N
    y, g = _pair(image, reference, window)
    loss3 = torch.empty(3, dtype=torch.float64, device=y.device)
    grad = torch.empty_like(y)
    N.call("rcgs_loss_grad_f64", N.ptr(y), N.ptr(g), int(y.shape[0]), int(y.shape[1]), float(lam),
           N.ptr(loss3), N.ptr(grad), D.stream_ptr())
    return loss3.cpu().numpy(), grad


def l1_loss(image, reference) -> float:
    return float(_run(image, reference, 0.0, False)[0][0])


def ssim(image, reference) -> float:
    return float(_run(image, reference, 0.0, True)[0][1])


def photometric_loss(image, reference, lam: float = DEFAULT_LAMBDA) -> LossBreakdown:
    """losses.py:95-101."""
    _lam(lam)
    l1, s, total = _run(image, reference, lam, True)[0]
    return LossBreakdown(l1=float(l1), ssim=float(s), total=float(total), lam=lam)


def loss_grad_wrt_image(image, reference, lam: float = DEFAULT_LAMBDA) -> np.ndarray:
    """d total / d image (H, W, 3) float64 (losses.py:118-134)."""
    _lam(lam)
    _, grad = _run(image, reference, lam, lam > 0.0)
    return grad.double().cpu().numpy()


def loss_and_grad_device(image: torch.Tensor, target: torch.Tensor, lam: float = DEFAULT_LAMBDA):
    """Device-resident variant used by the optimizer: (loss3 fp64, grad fp32)."""
    return D.loss_grad(image, target, lam)
