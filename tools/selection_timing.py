"""Selection-pass wall time per config, prefetched (views built ahead on worker
streams) vs inline (views kept), twice each: the first prefetched run in a
process pays a one-time thread/stream setup.

    python tools/selection_timing.py
"""
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2511_18441_b200 as P
from paper_2511_18441_b200 import device as D
torch.cuda.set_device(0)
for c in ("c1", "c2", "c3"):
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(bench.CONFIGS[c], 0, torch.device("cuda", 0))
    pts = D.to_device(cloud.points, torch.float64)
    for keep in (False, True, False, True):
        sp = P.SelectionPass(ds, cams, gt, keep_views=keep)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        sp.run(pts, (1.0, 0.2, 0.2))
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) * 1e3
        print(c, "inline(keep)" if keep else "prefetch", f"{dt:.1f} ms for {len(cams)} views")
