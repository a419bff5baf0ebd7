"""Golden stereo vectors from the REAL reference (`splattint.stereo`), SURVEY.md
8(f) row 3.  Run once in the build container:

    python tests/golden/make_stereo_golden.py

stereo_golden.npz:
  tex_*       textured pairs (reference test_stereo.py generator) with integer
              shifts, gray and colour, plus match_disparity outputs (max_disparity
              16 and a search wider than the image)
  plane_*     the reference's plane bundle view 0 (64x64 fronto-parallel at z=2.3,
              baseline 0.2): its float64 H/V stereo renders and the reference's
              match_disparity / stereo_hv_depth / estimate_depth outputs
"""

from __future__ import annotations

import os
import sys

import numpy as np
from scipy.ndimage import gaussian_filter

sys.path.insert(0, "/root/reference/pkg/src")
import splattint as st  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def textured(seed, size=48):
    rng = np.random.default_rng(seed)
    noise = gaussian_filter(rng.uniform(0.0, 1.0, (size, size)), sigma=1.2)
    return (noise - noise.min()) / (noise.max() - noise.min())


def main():
    out = {}
    cfg16 = st.StereoConfig(max_disparity=16)
    for k, shift in enumerate((0, 3, 7)):
        left = textured(10 + k)
        right = np.roll(left, -shift, axis=1)
        out[f"tex{k}_left"], out[f"tex{k}_right"] = left, right
        out[f"tex{k}_disp16"] = st.match_disparity(left, right, cfg16)
    # colour (non-gray) pair, different search / window settings
    rng = np.random.default_rng(4)
    col_l = np.stack([textured(20 + c, 40) for c in range(3)], axis=2)
    col_r = np.roll(col_l, -5, axis=1) * rng.uniform(0.9, 1.1, (1, 1, 3))
    out["col_left"], out["col_right"] = col_l, col_r
    cfg_c = st.StereoConfig(max_disparity=11, window_radius=3, lr_tolerance=0.5)
    out["col_disp"] = st.match_disparity(col_l, col_r, cfg_c)
    small = textured(7, 24)
    out["wide_img"] = small
    out["wide_disp"] = st.match_disparity(small, np.roll(small, -2, axis=1), st.StereoConfig(max_disparity=64))

    bundle = st.generate_synthetic_scene("plane", seed=0)
    intr = bundle.views[0].intrinsics
    pose = st.look_at((0.0, 0.0, -2.3), (0.0, 0.0, 0.0))
    cfg = st.StereoConfig(baseline=0.2)
    ph = st.render_stereo_pair(bundle.scene, intr, pose, 0.2, "horizontal")
    pv = st.render_stereo_pair(bundle.scene, intr, pose, 0.2, "vertical")
    out["plane_left"], out["plane_right_h"], out["plane_right_v"] = ph.left, ph.right, pv.right
    out["plane_disp_h"] = st.match_disparity(ph.left, ph.right, cfg)
    out["plane_disp_v"] = st.match_disparity(np.swapaxes(pv.left, 0, 1), np.swapaxes(pv.right, 0, 1), cfg).T
    out["plane_hv"] = st.stereo_hv_depth(bundle.scene, intr, pose, cfg)
    out["plane_est"] = st.estimate_depth(bundle.scene, intr, pose, "stereo-hv", config=cfg)
    out["plane_rot"], out["plane_t"] = pose.rotation, pose.translation
    out["plane_intr"] = np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height], np.float64)
    for f in ("positions", "rotations", "scales", "opacities", "sh"):
        out[f"plane_scene_{f}"] = getattr(bundle.scene, f)
    view = bundle.views[0]
    out["plane_v0_est"] = st.estimate_depth(bundle.scene, view.intrinsics, view.pose, "stereo-hv")
    out["plane_v0_rot"], out["plane_v0_t"] = view.pose.rotation, view.pose.translation
    np.savez_compressed(os.path.join(OUT, "stereo_golden.npz"), **out)
    for k, v in out.items():
        if k.endswith(("disp16", "disp", "disp_h", "disp_v")):
            print(k, v.shape, "valid", float((v >= 0).mean()))
    print("plane_hv finite", float(np.isfinite(out["plane_hv"]).mean()))


if __name__ == "__main__":
    main()
