"""One bracketed pass of the 8(f) rows for ncu: stereo-hv depth of a C3 view
(1M gaussians, 1080p) and the device PLY decode + encode of the C3 scene, each
warmed up once outside the cudaProfilerStart/Stop range.

    ncu --set full --profile-from-start off -k regex:"stereo_|ply_" python tools/extras_probe.py
"""

from __future__ import annotations

import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18441_b200 as P  # noqa: E402
from paper_2511_18441_b200 import scene_io as SIO  # noqa: E402
from paper_2511_18441_b200 import stereo as S  # noqa: E402


def main():
    torch.cuda.set_device(0)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(bench.CONFIGS["c3"], 0, torch.device("cuda", 0))
    intr, pose = cams[0]
    base = S.default_baseline(scene)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "c3.ply")
        P.save_scene_ply(scene, path)
        for bracket in (False, True):
            if bracket:
                torch.cuda.synchronize()
                torch.cuda.cudart().cudaProfilerStart()
            S.stereo_hv_depth_device(ds, sh0, intr, pose, base, backfill_tau=0.5)
            dsc, sh = P.load_scene_ply_device(path)
            SIO.save_scene_ply_device(scene, sh, os.path.join(tmp, "out.ply"))
            torch.cuda.synchronize()
            if bracket:
                torch.cuda.cudart().cudaProfilerStop()
            dsc.close()
    print("extras-probe ok")


if __name__ == "__main__":
    main()
