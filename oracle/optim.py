"""Float64 restatement of the SH backward, Adam and the refit iteration.

TEST INFRASTRUCTURE ONLY.  Follows backward.py:22-40 and optimize.py:59-120,
252-259 of /root/reference/pkg/src/splattint.  ``run_batched`` is the
schedule-driven restatement of the multi-GPU extension:
Adam(mean over the step's view batch of backward_sh(render_forward(v),
loss_grad(v))), which is the reference iteration exactly when the batch size
is 1.
"""

from __future__ import annotations

import numpy as np

from . import losses, raster
from .config import BETA1, BETA2, EPS, LAMBDA, LR_DC, LR_REST


def backward_sh(cap, grad_image):
    """dL/dSH (N, 16, 3) from a render_forward capture; backward.py:22-40."""
    p = cap["proj"]
    out = np.zeros((cap["n"], 16, 3))
    if p.count == 0 or cap["contrib_weight"].size == 0:
        return out
    flat = np.asarray(grad_image, np.float64).reshape(-1, 3)
    acc = np.zeros((p.count, 3))
    np.add.at(acc, cap["contrib_kept"], flat[cap["contrib_pixel"]] * cap["contrib_weight"][:, None])
    acc *= p.active
    out[p.index] = p.basis[:, :, None] * acc[:, None, :]
    return out


def adam(params, grads, m, v, step, lr_dc=LR_DC, lr_rest=LR_REST):
    """Bias-corrected Adam, optimize.py:59-83.  Returns (params, m, v, step,
    accepted); a non-finite gradient rejects the update."""
    if not np.all(np.isfinite(grads)):
        return params, m, v, step, False
    t = step + 1
    m = BETA1 * m + (1.0 - BETA1) * grads
    v = BETA2 * v + (1.0 - BETA2) * grads * grads
    mh = m / (1.0 - BETA1 ** t)
    vh = v / (1.0 - BETA2 ** t)
    lr = np.full((16, 1), lr_rest)
    lr[0] = lr_dc
    return params - lr * mh / (np.sqrt(vh) + EPS), m, v, t, True


class Scene:
    """Minimal duck-typed scene for the oracle."""

    def __init__(self, positions, rotations, scales, opacities, sh, sh_degree=3):
        self.positions = np.asarray(positions, np.float64)
        self.rotations = np.asarray(rotations, np.float64)
        self.scales = np.asarray(scales, np.float64)
        self.opacities = np.asarray(opacities, np.float64)
        self.sh = np.asarray(sh, np.float64)
        self.sh_degree = sh_degree

    def with_sh(self, sh):
        return Scene(self.positions, self.rotations, self.scales, self.opacities, sh,
                     self.sh_degree)


def view_grad(scene, intr, pose, target, lam=LAMBDA):
    """One view's render -> loss -> image grad -> SH grad (optimize.py:109-112)."""
    cap = raster.render_forward(scene, intr, pose)
    l1, ss, total = losses.photometric(cap["image"], target, lam)
    g = losses.loss_grad(cap["image"], target, lam)
    return backward_sh(cap, g), (l1, ss, total)


def view_acc(scene, intr, pose, target, lam=LAMBDA):
    """Per-gaussian channel sums acc[i, ch] = active * sum_p g[p, ch] w_ip (N, 3)
    of one view -- backward.py:36-39 before the basis expansion -- plus the loss."""
    cap = raster.render_forward(scene, intr, pose)
    loss = losses.photometric(cap["image"], target, lam)
    g = losses.loss_grad(cap["image"], target, lam)
    p = cap["proj"]
    acc = np.zeros((len(scene.positions), 3))
    if p.count and cap["contrib_weight"].size:
        part = np.zeros((p.count, 3))
        flat = g.reshape(-1, 3)
        np.add.at(part, cap["contrib_kept"], flat[cap["contrib_pixel"]] * cap["contrib_weight"][:, None])
        acc[p.index] = part * p.active
    return acc, loss


def expand_mean(scene, centers, accs):
    """(1/G) sum_v basis(dir_v) (x) acc_v -> (N, 16, 3) (the multi-view gradient)."""
    out = np.zeros((len(scene.positions), 16, 3))
    for c, a in zip(centers, accs):
        d = scene.positions - c
        d = d / np.linalg.norm(d, axis=1, keepdims=True)
        out += raster.sh_basis(d, scene.sh_degree)[:, :, None] * a[:, None, :]
    return out / len(accs)


def run_batched(scene, views, seed, steps, batch=1, lam=LAMBDA):
    """`steps` Adam iterations; each draws `batch` views from
    default_rng(seed).integers(len(views), size=batch) (== the reference's
    per-iteration rng.integers draw when batch == 1, optimize.py:106) and
    applies Adam to the mean gradient.  `views` is a list of
    (intr, pose, target).  Returns (scene, metrics list)."""
    rng = np.random.default_rng(seed)
    m = np.zeros_like(scene.sh)
    v = np.zeros_like(scene.sh)
    step = 0
    metrics = []
    for _ in range(steps):
        picks = rng.integers(len(views), size=batch) if batch > 1 else [int(rng.integers(len(views)))]
        total = np.zeros_like(scene.sh)
        for pk in picks:
            intr, pose, target = views[int(pk)]
            g, loss = view_grad(scene, intr, pose, target, lam)
            total += g
            metrics.append((step + 1, int(pk)) + loss)
        total /= len(picks)
        sh, m, v, step, _ = adam(scene.sh, total, m, v, step)
        scene = scene.with_sh(sh)
    return scene, metrics
