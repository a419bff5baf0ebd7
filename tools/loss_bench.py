"""Standalone timing of the optimizer's loss (rcgs_loss_grad, fp32) on a 1080p
frame pair: mean of CUDA-event timed launches after warm-up (L2 flushed between
launches)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_18441_b200 import device as D  # noqa: E402


def main():
    h, w, reps = 1080, 1920, 50
    rng = np.random.default_rng(0)
    img = torch.from_numpy(rng.uniform(0, 1, (h, w, 3)).astype(np.float32)).cuda()
    tgt = (img * 0.9 + 0.05).contiguous()
    loss3 = torch.empty(3, dtype=torch.float64, device="cuda")
    grad = torch.empty_like(img)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        D.loss_grad(img, tgt, 0.2, loss3, grad)
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        D.loss_grad(img, tgt, 0.2, loss3, grad)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) * 1e3)
    print(json.dumps({"us_mean": round(float(np.mean(times)), 1),
                      "us_p50": round(float(np.median(times)), 1), "loss": [float(v) for v in loss3.cpu()]}))


if __name__ == "__main__":
    main()
