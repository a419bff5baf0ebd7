"""SH-only backward (drop-in for splattint/backward.py:22-40) on the K6 kernel.

dL/dC[i, k, ch] = Y_k(dir_i) * active[i, ch] * sum_p dL/dy[p, ch] * w_ip.
The device capture of `render_forward` carries the binned view; the kernel
re-traverses it (bit-identical decisions to the forward) and reduces per
gaussian deterministically.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from . import device as D
from .errors import ValidationError


def backward_sh(capture, grad_image) -> np.ndarray:
    """(N, 16, 3) float64 gradient from a `render_forward` capture."""
    view = getattr(capture, "_view", None)
    if view is None:
        raise ValidationError("backward_sh needs a capture produced by this package's render_forward")
    grad_image = np.asarray(grad_image, dtype=np.float64)
    if grad_image.shape != capture.image.shape:
        raise ValidationError(
            f"gradient image shape {grad_image.shape} does not match render {capture.image.shape}")
    acc = view.backward(D.to_device(grad_image))
    out = torch.empty((view.scene.n, 16, 3), dtype=torch.float32, device=D.device())
    center = (N.c_double * 3)(*view.center)
    N.call("rcgs_sh_grad", view.scene.handle, N.ptr(acc), center, N.ptr(out), D.stream_ptr())
    return out.double().cpu().numpy()
