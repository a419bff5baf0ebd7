"""Float64 restatement of the photometric loss and its image gradient.

TEST INFRASTRUCTURE ONLY.  Follows /root/reference/pkg/src/splattint/losses.py;
the separable zero-padded correlation is scipy.ndimage.correlate1d exactly as
the reference calls it (losses.py:48-51).
"""

from __future__ import annotations

import numpy as np
from scipy.ndimage import correlate1d

from .config import LAMBDA, SSIM_C1, SSIM_C2, SSIM_SIGMA, SSIM_WINDOW


def window(size=SSIM_WINDOW, sigma=SSIM_SIGMA):
    """losses.py:41-45."""
    off = np.arange(size, dtype=np.float64) - size // 2
    k = np.exp(-(off ** 2) / (2.0 * sigma ** 2))
    return k / k.sum()


def filt(x, k):
    """losses.py:48-51."""
    return correlate1d(correlate1d(x, k, axis=0, mode="constant", cval=0.0),
                       k, axis=1, mode="constant", cval=0.0)


def ssim_terms(y, g, k):
    """losses.py:73-84."""
    mass = filt(np.ones(y.shape[:2]), k)[..., None]
    mu1 = filt(y, k) / mass
    mu2 = filt(g, k) / mass
    var1 = filt(y * y, k) / mass - mu1 * mu1
    var2 = filt(g * g, k) / mass - mu2 * mu2
    cov = filt(y * g, k) / mass - mu1 * mu2
    return (mass, mu1, mu2, 2.0 * mu1 * mu2 + SSIM_C1, 2.0 * cov + SSIM_C2,
            mu1 * mu1 + mu2 * mu2 + SSIM_C1, var1 + var2 + SSIM_C2)


def l1(y, g):
    return float(np.mean(np.abs(np.asarray(y, np.float64) - np.asarray(g, np.float64))))


def ssim(y, g):
    """losses.py:87-92."""
    _, _, _, a1, a2, b1, b2 = ssim_terms(np.asarray(y, np.float64), np.asarray(g, np.float64),
                                         window())
    return float(np.mean((a1 * a2) / (b1 * b2)))


def photometric(y, g, lam=LAMBDA):
    """losses.py:95-101 -> (l1, ssim, total)."""
    a, s = l1(y, g), ssim(y, g)
    return a, s, (1.0 - lam) * a + lam * (1.0 - s)


def ssim_grad(y, g, k):
    """losses.py:104-115."""
    mass, mu1, mu2, a1, a2, b1, b2 = ssim_terms(y, g, k)
    d_mu1 = 2.0 * (mu2 * a2) / (b1 * b2) - 2.0 * mu1 * a1 * a2 / (b1 * b1 * b2)
    d_var1 = -(a1 * a2) / (b1 * b2 * b2)
    d_cov = 2.0 * a1 / (b1 * b2)
    out = filt(d_mu1 / mass, k) + 2.0 * y * filt(d_var1 / mass, k) \
        - 2.0 * filt(d_var1 * mu1 / mass, k) + g * filt(d_cov / mass, k) \
        - filt(d_cov * mu2 / mass, k)
    return out / y.size


def loss_grad(y, g, lam=LAMBDA):
    """losses.py:118-134."""
    y = np.asarray(y, np.float64)
    g = np.asarray(g, np.float64)
    if np.array_equal(y, g):
        return np.zeros_like(y)
    out = (1.0 - lam) * np.sign(y - g) / y.size
    if lam > 0.0:
        out = out - lam * ssim_grad(y, g, window())
    return out
