"""Raw pinned host->device copy bandwidth for a 1080p fp32 HWC target (24.9 MB),
one stream and two concurrent streams.

    python tools/h2d_bw.py
"""

import torch

torch.cuda.set_device(0)
n = 1920 * 1080 * 3
src = [torch.randn(n).pin_memory() for _ in range(8)]
dst = [torch.empty(n, device="cuda") for _ in range(8)]
for nstreams in (1, 2):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(64):
            s = streams[i % nstreams]
            s.wait_event(e0) if i < nstreams else None
            with torch.cuda.stream(s):
                dst[i % 8].copy_(src[i % 8], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"{nstreams} stream(s): {64 * n * 4 / (ms / 1e3) / 1e9:.1f} GB/s ({ms / 64:.3f} ms per 24.9 MB)")
