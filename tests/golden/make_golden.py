"""Generate golden vectors from the REAL reference (`splattint`) in the build
container.  Run once here (``/root/reference`` exists only in this container);
the resulting ``tests/golden/*.npz`` travel with the repo and pin both the CPU
oracle (``oracle/``) and the CUDA path.

    python tests/golden/make_golden.py [small|c1|all]

Fixtures:
  two_blobs_32.npz   reference conftest bundle (two-blobs, 32x32, 2 cams, seed 1):
                     projection order, renders, depth, capture, selection ->
                     edited dataset, loss/grad, backward_sh, one Adam step and a
                     10-iteration BackgroundOptimizer(seed=7) trajectory.
  orbit_room_96.npz  orbit-room preset (140 gaussians, 96x96, 8 cams, seed 0):
                     renders + depth of views 0 and 3, projection order.
  scaled_small.npz   the scaled generator at N=3000, SH deg 3,
                     3 views at 80x48: arrays + reference render/depth of view 0.
  c1.npz             config 1 (10k gaussians, SH deg 0, 4 views at 256x256):
                     view-0 render + depth, selection cloud, masks of all views,
                     20-iteration trajectory (metrics + final DC row).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import splattint as st  # noqa: E402
from splattint.render import _project_scene  # noqa: E402
from splattint.synthetic import (_ball_arrays, _plane_arrays, _ring_cameras,  # noqa: E402
                                 _round_trip_float32, recipe)

OUT = os.path.dirname(os.path.abspath(__file__))


def ref_scaled_scene(n, sh_degree, seed=0):
    """orbit-room construction with grid_n = round(sqrt(N/2))
    plane gaussians + the rest as ball gaussians with scales x (40/count)^(1/3),
    rounded through float32; built with the reference's own helpers."""
    rng = np.random.default_rng(seed)
    g = int(round(np.sqrt(n / 2.0)))
    plane = _plane_arrays(recipe("orbit-room", grid_n=g), rng)
    nb = n - g * g
    ball = list(_ball_arrays(rng, (0.0, 0.0, -0.55), 0.28, nb))
    ball[2] = ball[2] * (40.0 / nb) ** (1.0 / 3.0)
    arrays = tuple(np.concatenate(f) for f in zip(plane, ball))
    return st.Scene(*_round_trip_float32(*arrays), sh_degree=sh_degree), g * g


def ref_cameras(width, height, count):
    rec = recipe("orbit-room", width=width, height=height, camera_count=count)
    return [(intr, st.look_at(eye, (0.0, 0.0, 0.0))) for intr, eye in _ring_cameras(rec)]


def scene_dict(scene, prefix=""):
    return {prefix + "positions": scene.positions, prefix + "rotations": scene.rotations,
            prefix + "scales": scene.scales, prefix + "opacities": scene.opacities,
            prefix + "sh": scene.sh, prefix + "sh_degree": np.int64(scene.sh_degree)}


def cam_dict(intr, pose, prefix):
    return {prefix + "K": np.array([intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height],
                                   np.float64),
            prefix + "R": pose.rotation, prefix + "t": pose.translation}


def one_blob_cloud(bundle, first=10, radius=8.0):
    """test_acceptance.py:64-77 selection recipe."""
    view = bundle.views[0]
    centroid = bundle.scene.positions[:first].mean(axis=0)
    cam = view.pose.rotation @ centroid + view.pose.translation
    u = view.intrinsics.fx * cam[0] / cam[2] + view.intrinsics.cx
    v = view.intrinsics.fy * cam[1] / cam[2] + view.intrinsics.cy
    mask = st.apply_stroke(st.new_mask(view.intrinsics, view.pose), "brush",
                           [(float(u), float(v))], radius=radius)
    depth = st.depth_from_gaussians(bundle.scene, view.intrinsics, view.pose)
    cloud = st.unproject(mask, depth, fraction=0.7, seed=0)
    return mask.bits, st.remove_outliers(cloud, k=16, std_scale=0.007)


def make_two_blobs():
    bundle = st.generate_synthetic_scene(recipe("two-blobs", width=32, height=32,
                                                camera_count=2), seed=1)
    d = scene_dict(bundle.scene)
    for i, view in enumerate(bundle.views):
        d.update(cam_dict(view.intrinsics, view.pose, f"v{i}_"))
        d[f"v{i}_image"] = view.image
        d[f"v{i}_depth"] = st.depth_from_gaussians(bundle.scene, view.intrinsics, view.pose)
        proj = _project_scene(bundle.scene, view.intrinsics, view.pose)
        d[f"v{i}_order"] = proj.index
        d[f"v{i}_zsorted"] = proj.depth
        d[f"v{i}_mean2d"] = proj.mean2d
        d[f"v{i}_render_bg"] = st.render(bundle.scene, view.intrinsics, view.pose,
                                         background=(0.15, 0.05, 0.25))
    brush, cloud = one_blob_cloud(bundle)
    d["brush"] = brush
    d["cloud"] = cloud.points
    ds = st.build_edited_dataset(bundle.views, cloud, (1.0, 0.2, 0.2), bundle.scene)
    for i, ev in enumerate(ds.views):
        d[f"v{i}_mask"] = ev.mask
        d[f"v{i}_edited"] = ev.image
    # one optimizer step on fixed inputs (view 0)
    view = bundle.views[0]
    cap = st.render_forward(bundle.scene, view.intrinsics, view.pose)
    target = ds.views[0].image
    loss = st.photometric_loss(cap.image, target)
    grad_img = st.loss_grad_wrt_image(cap.image, target)
    grads = st.backward_sh(cap, grad_img)
    new_sh, state = st.adam_step(bundle.scene.sh, grads, st.AdamState.fresh(len(bundle.scene)))
    d.update(cap_image=cap.image, cap_kept_index=cap.kept_index, cap_pixel=cap.contrib_pixel,
             cap_kept=cap.contrib_kept, cap_weight=cap.contrib_weight, cap_active=cap.active,
             cap_basis=cap.basis, loss=np.array([loss.l1, loss.ssim, loss.total]),
             grad_image=grad_img, grads=grads, adam_sh=new_sh, adam_m=state.m, adam_v=state.v)
    # a target with a different sign field everywhere (criterion-1 style)
    target2 = np.clip(view.image * np.array([0.7, 0.2, 0.4]), 0.0, 1.0)
    d["target2"] = target2
    d["grad_image2"] = st.loss_grad_wrt_image(cap.image, target2)
    d["loss2"] = np.array(list(vars(st.photometric_loss(cap.image, target2)).values())[:3])
    d["grads2"] = st.backward_sh(cap, d["grad_image2"])
    # 10-iteration deterministic trajectory
    lines = []
    opt = st.BackgroundOptimizer(bundle.scene, ds, seed=7,
                                 metrics_sink=lambda m: lines.append(m.line()))
    final = opt.run_iterations(10)
    d["traj_lines"] = np.array(lines)
    d["traj_sh"] = final.sh
    np.savez_compressed(os.path.join(OUT, "two_blobs_32.npz"), **d)


def make_orbit_room():
    bundle = st.generate_synthetic_scene("orbit-room", seed=0)
    d = scene_dict(bundle.scene)
    for i in (0, 3):
        view = bundle.views[i]
        d.update(cam_dict(view.intrinsics, view.pose, f"v{i}_"))
        d[f"v{i}_image"] = view.image
        d[f"v{i}_depth"] = st.depth_from_gaussians(bundle.scene, view.intrinsics, view.pose)
        d[f"v{i}_order"] = _project_scene(bundle.scene, view.intrinsics, view.pose).index
    np.savez_compressed(os.path.join(OUT, "orbit_room_96.npz"), **d)


def make_scaled_small():
    scene, n_plane = ref_scaled_scene(3000, 3, seed=0)
    cams = ref_cameras(80, 48, 3)
    d = scene_dict(scene)
    d["n_plane"] = np.int64(n_plane)
    for i, (intr, pose) in enumerate(cams):
        d.update(cam_dict(intr, pose, f"v{i}_"))
    intr, pose = cams[0]
    d["v0_image"] = st.render(scene, intr, pose)
    d["v0_depth"] = st.depth_from_gaussians(scene, intr, pose)
    d["v0_order"] = _project_scene(scene, intr, pose).index
    np.savez_compressed(os.path.join(OUT, "scaled_small.npz"), **d)


def make_c1(steps=20):
    t0 = time.time()
    scene, n_plane = ref_scaled_scene(10_000, 0, seed=0)
    cams = ref_cameras(256, 256, 4)
    views = []
    for i, (intr, pose) in enumerate(cams):
        views.append(st.TrainingView(view_id=i, intrinsics=intr, pose=pose,
                                     image=st.render(scene, intr, pose)))
        print(f"c1: GT view {i} rendered at {time.time() - t0:.0f}s", flush=True)
    view = views[0]
    centroid = scene.positions[n_plane:].mean(axis=0)
    cam = view.pose.rotation @ centroid + view.pose.translation
    u = view.intrinsics.fx * cam[0] / cam[2] + view.intrinsics.cx
    v = view.intrinsics.fy * cam[1] / cam[2] + view.intrinsics.cy
    mask = st.apply_stroke(st.new_mask(view.intrinsics, view.pose), "brush",
                           [(float(u), float(v))], radius=0.15 * view.intrinsics.width)
    depth0 = st.depth_from_gaussians(scene, view.intrinsics, view.pose)
    cloud = st.remove_outliers(st.unproject(mask, depth0, fraction=0.7, seed=0),
                               k=16, std_scale=0.007)
    ds = st.build_edited_dataset(views, cloud, (1.0, 0.2, 0.2), scene)
    print(f"c1: dataset built at {time.time() - t0:.0f}s", flush=True)
    d = {"n": np.int64(10_000), "n_plane": np.int64(n_plane), "brush": mask.bits,
         "brush_uv": np.array([u, v]), "cloud": cloud.points, "v0_image": views[0].image,
         "v0_depth": depth0}
    for i, ev in enumerate(ds.views):
        d[f"v{i}_mask"] = ev.mask
    lines = []
    opt = st.BackgroundOptimizer(scene, ds, seed=7, metrics_sink=lambda m: lines.append(m.line()))
    final = opt.run_iterations(steps)
    d["traj_lines"] = np.array(lines)
    d["traj_dc"] = final.sh[:, 0, :]
    d["final_v0_render"] = st.render(final, views[0].intrinsics, views[0].pose).astype(np.float32)
    print(f"c1: trajectory done at {time.time() - t0:.0f}s", flush=True)
    np.savez_compressed(os.path.join(OUT, "c1.npz"), **d)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what in ("small", "all"):
        make_two_blobs()
        make_orbit_room()
        make_scaled_small()
    if what in ("c1", "all"):
        make_c1()
