import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2511_18441_b200 as P
from paper_2511_18441_b200 import device as D
torch.cuda.set_device(0)
for cfgname in ("c3",):
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(bench.CONFIGS[cfgname], 0, torch.device("cuda", 0))
    mx = []
    for i in range(0, len(cams), max(1, len(cams) // 8)):
        v = D.View(ds, cams[i][0], cams[i][1], P.DEFAULT_CONFIG)
        r = v.ranges().view(-1, 2).cpu().numpy().astype(np.int64)
        L = r[:, 1] - r[:, 0]
        mx.append((int(L.max()), int(np.percentile(L, 99)), float(L.mean()), int((L > 2048).sum()), int((L > 4096).sum()), v.n_pairs))
        v.close()
    print(cfgname, mx)
