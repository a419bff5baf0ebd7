"""GPU parity: the CUDA path (through the C ABI) against the reference golden
vectors and the CPU oracle on the same inputs.

Bars (north_star): depth orders, masks, kept sets and hit counts
bit-exact; images max abs <= 1e-4 per channel and PSNR > 60 dB; one optimizer
step on identical inputs within 1e-6; float tolerances are written per test.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_camera, identity_camera, make_scene

pytestmark = pytest.mark.gpu

import paper_2511_18441_b200 as P  # noqa: E402
from oracle import losses as OL, optim as OO, raster as OR, selection as OS  # noqa: E402

IMG_TOL = 1e-4


def psnr(a, b):
    mse = float(np.mean((np.asarray(a) - np.asarray(b)) ** 2))
    return np.inf if mse == 0 else 10 * np.log10(1.0 / mse)


def p_scene(d):
    return P.Scene(d["positions"], d["rotations"], d["scales"], d["opacities"], d["sh"], int(d["sh_degree"]))


def p_cam(d, prefix):
    intr, pose = golden_camera(d, prefix)
    return (P.CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height),
            P.CameraPose(pose.rotation, pose.translation))


def p_from_ns(ns):
    return P.Scene(ns.positions, ns.rotations, ns.scales, ns.opacities, ns.sh, ns.sh_degree)


def p_cam_ns(intr, pose):
    return (P.CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height),
            P.CameraPose(pose.rotation, pose.translation))


def assert_image_close(img, ref, tol=IMG_TOL):
    diff = np.abs(img - ref)
    assert diff.max() <= tol, f"max abs {diff.max():.3e} (PSNR {psnr(img, ref):.1f} dB)"
    assert psnr(img, ref) > 60.0


def assert_depth_exact(dep, ref):
    np.testing.assert_array_equal(np.isfinite(dep), np.isfinite(ref))
    np.testing.assert_array_equal(dep[np.isfinite(dep)], ref[np.isfinite(ref)])


# ---------------------------------------------------------------- preprocess + sort
@pytest.mark.parametrize("fixture,views", [("two_blobs", (0, 1)), ("orbit_room", (0, 3)),
                                            ("scaled_small", (0,))])
def test_kept_order_bit_exact(fixture, views, request):
    from paper_2511_18441_b200 import device as D
    d = request.getfixturevalue(fixture)
    scene = p_scene(d)
    for v in views:
        intr, pose = p_cam(d, f"v{v}_")
        view = D.View(D.device_scene(scene), intr, pose, P.DEFAULT_CONFIG)
        idx, z = view.kept()
        np.testing.assert_array_equal(idx.cpu().numpy(), d[f"v{v}_order"])
        np.testing.assert_array_equal(z.cpu().numpy(), OR.project(scene, intr, pose).depth)


@pytest.mark.parametrize("run", [6, 40])
def test_depth_order_near_ties_bit_exact(run):
    """Depths equal in their top 32 varying key bits but decreasing with scene
    index: a short run is repaired in place, a run longer than 32 takes the
    full 64-bit sort path; both must give np.argsort(z, kind="stable")."""
    from paper_2511_18441_b200 import device as D
    rng = np.random.default_rng(run)
    spread = [dict(position=(rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), rng.uniform(1.0, 7.0)), scale=0.05)
              for _ in range(200)]
    ties = [dict(position=(rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), 3.0 + 1e-13 * (run - i)), scale=0.05)
            for i in range(run)]
    exact = [dict(position=(0.1 * i - 0.2, 0.05, 2.5), scale=0.05) for i in range(5)]  # identical z
    ns = make_scene(spread[:100] + ties + exact + spread[100:])
    scene = p_from_ns(ns)
    intr, pose = p_cam_ns(*identity_camera(64, 64, fx=64.0))
    view = D.View(D.device_scene(scene), intr, pose, P.DEFAULT_CONFIG)
    idx, z = view.kept()
    np.testing.assert_array_equal(idx.cpu().numpy(), OR.project(ns, intr, pose).index)


# ---------------------------------------------------------------- raster + depth
@pytest.mark.parametrize("fixture,views", [("two_blobs", (0, 1)), ("orbit_room", (0, 3)),
                                            ("scaled_small", (0,))])
def test_render_and_depth_match_reference(fixture, views, request):
    d = request.getfixturevalue(fixture)
    scene = p_scene(d)
    for v in views:
        intr, pose = p_cam(d, f"v{v}_")
        assert_image_close(P.render(scene, intr, pose), d[f"v{v}_image"])
        assert_depth_exact(P.depth_from_gaussians(scene, intr, pose), d[f"v{v}_depth"])


def test_background_and_layout(two_blobs):
    scene = p_scene(two_blobs)
    intr, pose = p_cam(two_blobs, "v0_")
    assert_image_close(P.render(scene, intr, pose, background=(0.15, 0.05, 0.25)), two_blobs["v0_render_bg"])
    hwc = P.render(scene, intr, pose)
    np.testing.assert_array_equal(P.render(scene, intr, pose, layout="chw"), P.to_chw(hwc))
    with pytest.raises(P.ValidationError):
        P.render(scene, intr, pose, layout="hcw")


def test_capture_matches_reference(two_blobs):
    scene = p_scene(two_blobs)
    intr, pose = p_cam(two_blobs, "v0_")
    cap = P.render_forward(scene, intr, pose)
    np.testing.assert_array_equal(cap.contrib_pixel, two_blobs["cap_pixel"])
    np.testing.assert_array_equal(cap.contrib_kept, two_blobs["cap_kept"])
    np.testing.assert_allclose(cap.contrib_weight, two_blobs["cap_weight"], atol=1e-6)
    np.testing.assert_array_equal(cap.kept_index, two_blobs["cap_kept_index"])
    np.testing.assert_array_equal(cap.active, two_blobs["cap_active"])
    np.testing.assert_allclose(cap.basis, two_blobs["cap_basis"], atol=1e-15)
    # weight budget: sum_i w + T_final == 1 per pixel (test_render.py:221-234)
    ws = np.zeros(intr.width * intr.height)
    np.add.at(ws, cap.contrib_pixel, cap.contrib_weight)
    white = P.render(scene, intr, pose, background=(1.0, 1.0, 1.0))
    np.testing.assert_allclose(ws.reshape(intr.height, intr.width) + (white - cap.image)[:, :, 0], 1.0,
                               atol=1e-5)


def test_known_answers():
    intr, pose = p_cam_ns(*identity_camera(33, 33, fx=40.0))
    two = p_from_ns(make_scene([dict(position=(0, 0, 1.0), color=(1, 0, 0), opacity=0.5),
                                dict(position=(0, 0, 2.0), color=(0, 0, 1), opacity=0.9995)]))
    np.testing.assert_allclose(P.render(two, intr, pose)[16, 16], [0.5, 0.0, 0.495], atol=1e-6)
    one = p_from_ns(make_scene([dict(position=(0, 0, 1.0), color=(1, 0, 0), opacity=0.25)]))
    np.testing.assert_allclose(P.render(one, intr, pose, background=(0, 1, 0))[16, 16], [0.25, 0.75, 0.0],
                               atol=1e-6)
    strict = p_from_ns(make_scene([dict(position=(0, 0, 1.0), opacity=0.5)]))
    assert np.isinf(P.depth_from_gaussians(strict, intr, pose)[16, 16])
    twod = p_from_ns(make_scene([dict(position=(0, 0, 1.0), opacity=0.4),
                                 dict(position=(0, 0, 2.0), opacity=0.4)]))
    assert P.depth_from_gaussians(twod, intr, pose)[16, 16] == 2.0
    behind = p_from_ns(make_scene([dict(position=(0, 0, -3.0))]))
    np.testing.assert_array_equal(P.render(behind, intr, pose), 0.0)
    empty = P.Scene(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 16, 3)))
    np.testing.assert_array_equal(P.render(empty, intr, pose, background=(0.2, 0.4, 0.6)),
                                  np.broadcast_to((0.2, 0.4, 0.6), (33, 33, 3)))
    assert np.all(np.isinf(P.depth_from_gaussians(empty, intr, pose)))


def test_random_scenes_match_oracle():
    """Ragged image sizes, anisotropic gaussians, near-clip and off-screen cases."""
    rng = np.random.default_rng(11)
    for trial, (w, h) in enumerate([(17, 9), (40, 23), (64, 64), (31, 50)]):
        specs = []
        for _ in range(60):
            q = rng.normal(size=4)
            specs.append(dict(position=rng.uniform(-0.9, 0.9, 3) + [0, 0, 2.0],
                              color=rng.uniform(0.0, 1.0, 3), scale=rng.uniform(0.01, 0.3, 3),
                              opacity=rng.uniform(0.02, 0.99), quat=q / np.linalg.norm(q)))
        # near-clip cases (render.py:176: kept iff z > 0.2) and very close large footprints
        for z in (0.2, 0.2001, np.nextafter(0.2, 1.0), 0.23, 0.35):
            specs.append(dict(position=(rng.uniform(-0.05, 0.05), rng.uniform(-0.05, 0.05), z),
                              color=rng.uniform(0.0, 1.0, 3), scale=rng.uniform(0.002, 0.02, 3),
                              opacity=rng.uniform(0.3, 0.99), quat=(1.0, 0.0, 0.0, 0.0)))
        ns = make_scene(specs)
        ns.sh[:, 1:, :] = rng.normal(0, 0.2, (len(specs), 15, 3))
        scene = p_from_ns(ns)
        intr, pose = p_cam_ns(*identity_camera(w, h, fx=float(max(w, h))))
        assert_image_close(P.render(scene, intr, pose), OR.render(ns, intr, pose))
        assert_depth_exact(P.depth_from_gaussians(scene, intr, pose), OR.depth(ns, intr, pose))


# ---------------------------------------------------------------- loss / backward / adam
def _f32(x):
    return np.asarray(x, np.float32).astype(np.float64)


def test_loss_and_grad_match_oracle(two_blobs):
    image, target = _f32(two_blobs["cap_image"]), _f32(two_blobs["v0_edited"])
    lb = P.photometric_loss(image, target)
    l1, ss, total = OL.photometric(image, target)
    assert abs(lb.l1 - l1) < 1e-12 and abs(lb.ssim - ss) < 1e-12 and abs(lb.total - total) < 1e-12
    for tgt in (target, _f32(two_blobs["target2"])):
        g = P.loss_grad_wrt_image(image, tgt)
        ref = OL.loss_grad(image, tgt)
        # relative to the gradient scale; where y == gt the reference itself only
        # leaves round-off residue (~1e-20) whose sign is arbitrary
        assert np.abs(g - ref).max() <= 1e-6 * np.abs(ref).max()
    np.testing.assert_array_equal(P.loss_grad_wrt_image(image, image), 0.0)
    small_y, small_g = np.zeros((4, 4, 3)), np.ones((4, 4, 3))
    np.testing.assert_array_equal(P.loss_grad_wrt_image(small_y, small_g, lam=0.0), -np.ones((4, 4, 3)) / 48)
    with pytest.raises(P.ValidationError):
        P.loss_grad_wrt_image(small_y, small_g, lam=0.2)


def test_loss_grad_local_differences_match_oracle():
    """Differences confined to small patches (one straddling a 32-px block corner):
    the block-sparse loss kernels must equal the dense oracle everywhere."""
    rng = np.random.default_rng(21)
    img = rng.uniform(0.1, 0.9, (150, 170, 3))
    tgt = img.copy()
    tgt[28:35, 29:36] = np.clip(tgt[28:35, 29:36] * [1.0, 0.3, 0.3], 0, 1)   # block corner (32, 32)
    tgt[120:124, 140:150, 1] += 0.05
    for lam in (0.2, 0.0):
        g = P.loss_grad_wrt_image(img, tgt, lam=lam)
        ref = OL.loss_grad(img, tgt, lam=lam)
        assert np.abs(g - ref).max() <= 1e-9 * np.abs(ref).max()
        # beyond one 32-px block of any difference the gradient is an exact zero
        # (the dense formula leaves ~1e-20 round-off there)
        far = np.ones(img.shape[:2], bool)
        far[:96, :96] = False
        far[64:, 96:] = False
        assert np.all(g[far] == 0.0)
    lb = P.photometric_loss(img, tgt)
    l1, ss, total = OL.photometric(img, tgt)
    assert abs(lb.l1 - l1) < 1e-13 and abs(lb.ssim - ss) < 1e-12 and abs(lb.total - total) < 1e-12


def _window_clean(img, tgt, radius):
    """True where the (2 radius + 1)^2 window (zero padded) has img == tgt everywhere."""
    from scipy.ndimage import maximum_filter
    diff = np.any(img != tgt, axis=2).astype(np.uint8)
    return maximum_filter(diff, size=2 * radius + 1, mode="constant", cval=0) == 0


@pytest.mark.parametrize("shape", [(150, 170), (37, 300), (11, 11), (205, 64), (131, 129)])
def test_device_loss_fp32_matches_oracle(shape):
    """The optimizer's loss (rcgs_loss_grad: fp32 images and gradient, fp32
    gradient maps between the passes) against the fp64 oracle: loss terms within
    1e-12, gradient within 1e-6 of its scale; where the 21x21 window has no
    difference the gradient is zero up to the reference's own round-off residue
    (exactly zero beyond one 32-px block of a difference), and identical images
    give (0, 1, 0) and an all-zero gradient."""
    import torch
    from paper_2511_18441_b200 import device as D
    rng = np.random.default_rng(shape[0] * 1000 + shape[1])
    h, w = shape
    img = rng.uniform(0.05, 0.95, (h, w, 3)).astype(np.float32)
    tgt = img.copy()
    # local edits (one straddling strip / band boundaries) plus a region of noise
    tgt[h // 3:h // 3 + 7, w // 2 - 3:w // 2 + 4] *= np.float32(0.4)
    tgt[-5:, -9:, 1] = np.clip(tgt[-5:, -9:, 1] + 0.1, 0, 1)
    tgt[:3, :4, 2] = 0.0
    for lam in (0.2, 0.0):
        y_d = torch.from_numpy(img).cuda()
        g_d = torch.from_numpy(tgt).cuda()
        loss3, grad = D.loss_grad(y_d, g_d, lam)
        l1, ss, total = (float(v) for v in loss3.cpu())
        y64, g64 = img.astype(np.float64), tgt.astype(np.float64)
        rl1, rss, rtotal = OL.photometric(y64, g64, lam=lam)
        assert abs(l1 - rl1) < 1e-12 and abs(ss - rss) < 1e-12 and abs(total - rtotal) < 1e-12
        ref = OL.loss_grad(y64, g64, lam=lam)
        gd = grad.double().cpu().numpy()
        assert np.abs(gd - ref).max() <= 1e-6 * np.abs(ref).max()
        if lam > 0:
            clean = _window_clean(img, tgt, 10)
            assert np.all(np.abs(ref[clean]) < 1e-15)
            assert np.all(np.abs(gd[clean]) < 1e-15)
    same = torch.from_numpy(img).cuda()
    loss3, grad = D.loss_grad(same, same.clone(), 0.2)
    assert [float(v) for v in loss3.cpu()] == [0.0, 1.0, 0.0]
    assert torch.count_nonzero(grad).item() == 0


def test_device_loss_fp32_full_hd_sampled():
    """1080p (the C3 frame): fp32 fused loss vs the fp64 oracle on the whole frame
    (loss terms) and the gradient everywhere."""
    import torch
    from paper_2511_18441_b200 import device as D
    rng = np.random.default_rng(3)
    h, w = 1080, 1920
    img = rng.uniform(0.0, 1.0, (h, w, 3)).astype(np.float32)
    tgt = img.copy()
    tgt[200:700, 300:1500] = np.clip(tgt[200:700, 300:1500] * np.float32(0.7) + np.float32(0.1), 0, 1)
    tgt[900:, :, 0] = rng.uniform(0.0, 1.0, (h - 900, w)).astype(np.float32)
    loss3, grad = D.loss_grad(torch.from_numpy(img).cuda(), torch.from_numpy(tgt).cuda(), 0.2)
    y64, g64 = img.astype(np.float64), tgt.astype(np.float64)
    rl1, rss, rtotal = OL.photometric(y64, g64)
    l1, ss, total = (float(v) for v in loss3.cpu())
    assert abs(l1 - rl1) < 1e-12 and abs(ss - rss) < 1e-12 and abs(total - rtotal) < 1e-12
    ref = OL.loss_grad(y64, g64)
    gd = grad.double().cpu().numpy()
    assert np.abs(gd - ref).max() <= 1e-6 * np.abs(ref).max()
    clean = _window_clean(img, tgt, 10)
    assert clean.any() and np.all(np.abs(gd[clean]) < 1e-15)


def test_backward_matches_oracle(two_blobs):
    scene = p_scene(two_blobs)
    intr, pose = p_cam(two_blobs, "v0_")
    cap = P.render_forward(scene, intr, pose)
    ocap = OR.render_forward(scene, intr, pose)
    for key in ("grad_image", "grad_image2"):
        g = _f32(two_blobs[key])
        grads = P.backward_sh(cap, g)
        ref = OO.backward_sh(ocap, g)
        assert np.abs(grads - ref).max() <= 1e-6 * np.abs(ref).max() + 1e-15
    # culled gaussians and inactive channels get exactly zero
    mask = np.ones(len(scene), bool)
    mask[cap.kept_index] = False
    assert np.all(grads[mask] == 0.0)


def test_adam_matches_oracle(two_blobs):
    grads = two_blobs["grads"]
    sh = two_blobs["sh"]
    new_sh, state = P.adam_step(sh, grads, P.AdamState.fresh(len(sh)))
    np.testing.assert_allclose(new_sh, two_blobs["adam_sh"], atol=1e-6)
    assert state.step == 1
    same, st = P.adam_step(sh, np.zeros_like(sh), P.AdamState.fresh(len(sh)))
    np.testing.assert_array_equal(same, sh)
    bad = grads.copy()
    bad[1, 3, 2] = np.nan
    s0 = P.AdamState.fresh(len(sh))
    out, s1 = P.adam_step(sh, bad, s0)
    assert out is sh and s1 is s0


def test_fused_step_matches_oracle_one_iteration(two_blobs):
    """optimize_iteration on the device vs the oracle's iteration on the same
    scene, view and (float32) target: |d theta| <= 1e-6."""
    scene = p_scene(two_blobs)
    views = []
    for v in (0, 1):
        intr, pose = p_cam(two_blobs, f"v{v}_")
        views.append(P.TrainingView(v, intr, pose, _f32(two_blobs[f"v{v}_image"])))
    ev = tuple(P.EditedView(view=vw, mask=two_blobs[f"v{i}_mask"], image=_f32(two_blobs[f"v{i}_edited"]))
               for i, vw in enumerate(views))
    ds = P.EditedDataset(views=ev, generation=0, tint=np.array([1.0, 0.2, 0.2]))
    rng = np.random.default_rng(7)
    new_scene, state, metrics = P.optimize_iteration(scene, ds, rng, P.AdamState.fresh(len(scene)))
    pick = int(np.random.default_rng(7).integers(2))
    assert metrics.view_id == pick and metrics.iteration == 1
    intr, pose = p_cam(two_blobs, f"v{pick}_")
    # oracle on the float32-rounded image the device renders
    img = P.render(scene, intr, pose)
    tgt = ev[pick].image
    ocap = OR.render_forward(scene, intr, pose)
    g = OL.loss_grad(img, tgt)
    grads = OO.backward_sh(ocap, g)
    ref_sh, *_ = OO.adam(scene.sh, grads, np.zeros_like(grads), np.zeros_like(grads), 0)
    assert np.abs(new_scene.sh - ref_sh).max() <= 1e-6
    np.testing.assert_array_equal(new_scene.positions, scene.positions)


# ---------------------------------------------------------------- selection pass
def test_project_cloud_and_dataset_bit_exact(two_blobs):
    scene = p_scene(two_blobs)
    views = []
    for v in (0, 1):
        intr, pose = p_cam(two_blobs, f"v{v}_")
        views.append(P.TrainingView(v, intr, pose, two_blobs[f"v{v}_image"]))
        dep = P.depth_from_gaussians(scene, intr, pose)
        mask = P.project_cloud(P.SelectionCloud(two_blobs["cloud"]), intr, pose, dep)
        np.testing.assert_array_equal(mask, two_blobs[f"v{v}_mask"])
    ds = P.build_edited_dataset(views, P.SelectionCloud(two_blobs["cloud"]), (1.0, 0.2, 0.2), scene)
    for v, ev in enumerate(ds.views):
        np.testing.assert_array_equal(ev.mask, two_blobs[f"v{v}_mask"])
        np.testing.assert_array_equal(ev.image, two_blobs[f"v{v}_edited"])
    empty = P.build_edited_dataset(views, P.empty_cloud(), (0.1, 0.1, 0.1), scene, generation=5)
    assert empty.generation == 5 and not any(ev.mask.any() for ev in empty.views)


def test_project_cloud_known_answers():
    intr, pose = p_cam_ns(*identity_camera(33, 33))
    occ = np.full((33, 33), 1.0)
    bits = P.project_cloud(P.SelectionCloud(np.array([[0.0, 0.0, 1.0]])), intr, pose, occ)
    assert bits[14:19, 14:19].all() and bits.sum() == 25
    assert P.project_cloud(P.SelectionCloud(np.array([[0.0, 0.0, 1.02]])), intr, pose, occ).any()
    assert not P.project_cloud(P.SelectionCloud(np.array([[0.0, 0.0, 1.0201]])), intr, pose, occ).any()
    b = P.project_cloud(P.SelectionCloud(np.array([[-0.5, -0.5, 1.0]])), intr, pose, np.full((33, 33), 10.0))
    assert b[:3, :3].all() and b.sum() == 9
    assert P.project_cloud(P.SelectionCloud(np.array([[0.0, 0.0, -1.0]])), intr, pose,
                           np.full((33, 33), 10.0)).sum() == 0
    out = P.apply_recolor(np.full((1, 1, 3), [0.9, 0.3, 0.6]), np.ones((1, 1), bool), (2.0, 2.0, 2.0))
    np.testing.assert_array_equal(out[0, 0], [1.0, 0.6, 1.0])


def test_random_cloud_masks_bit_exact(orbit_room):
    scene = p_scene(orbit_room)
    rng = np.random.default_rng(5)
    pts = rng.uniform(-1.0, 1.0, (5000, 3)) * [1, 1, 0.6]
    for v in (0, 3):
        intr, pose = p_cam(orbit_room, f"v{v}_")
        dep = orbit_room[f"v{v}_depth"]
        for quad in (1, 4, 5):
            np.testing.assert_array_equal(P.project_cloud(P.SelectionCloud(pts), intr, pose, dep, quad),
                                          OS.project_cloud(pts, intr, pose, dep, quad))


def test_selection_pass_mask_hits_exact(two_blobs):
    import torch
    from paper_2511_18441_b200 import device as D
    scene = p_scene(two_blobs)
    cams = [p_cam(two_blobs, f"v{v}_") for v in (0, 1)]
    gt = torch.stack([D.to_device(two_blobs[f"v{v}_image"]) for v in (0, 1)])
    sp = P.SelectionPass(D.device_scene(scene), cams, gt)
    sp.run(D.to_device(two_blobs["cloud"], torch.float64), (1.0, 0.2, 0.2))
    masks = sp.masks.cpu().numpy().astype(bool)
    for v in (0, 1):
        np.testing.assert_array_equal(masks[v], two_blobs[f"v{v}_mask"])
    hits, wsum = OS.mask_hits(scene, cams, [two_blobs["v0_mask"], two_blobs["v1_mask"]])
    np.testing.assert_array_equal(sp.hits.cpu().numpy(), hits)
    np.testing.assert_allclose(sp.wsum_float().cpu().numpy(), wsum, atol=1e-5)
    np.testing.assert_allclose(sp.edited.cpu().numpy(), _f32(np.stack([two_blobs["v0_edited"], two_blobs["v1_edited"]])),
                               atol=1e-7)


def test_selection_pass_prefetched_equals_inline(orbit_room):
    """SelectionPass builds upcoming views on worker streams when it does not keep
    them; masks, edited targets, hit counts and weights equal the inline path's."""
    import torch
    from paper_2511_18441_b200 import device as D
    scene = p_scene(orbit_room)
    cams = [p_cam(orbit_room, f"v{v}_") for v in (0, 3)] * 4  # 8 views
    ds = D.device_scene(scene)
    gt = torch.stack([D.to_device(orbit_room[f"v{v}_image"]) for v in (0, 3)] * 4)
    rng = np.random.default_rng(9)
    pts = D.to_device(rng.uniform(-1.0, 1.0, (4000, 3)) * [1, 1, 0.6], torch.float64)
    a = P.SelectionPass(ds, cams, gt).run(pts, (1.0, 0.2, 0.2))            # prefetched
    b = P.SelectionPass(ds, cams, gt, keep_views=True).run(pts, (1.0, 0.2, 0.2))  # inline
    assert torch.equal(a.masks, b.masks) and torch.equal(a.edited, b.edited)
    assert torch.equal(a.hits, b.hits) and torch.equal(a.wsum, b.wsum)
    assert int(a.masks.sum()) > 0


# ---------------------------------------------------------------- optimizer trajectory
def test_refit_trajectory_tracks_reference(two_blobs):
    """10 iterations of BackgroundOptimizer(seed=7) vs the reference run.  The
    view sequence is identical (same RNG stream); losses track the reference
    within the fp32 trajectory tolerance of SURVEY.md 0.7."""
    scene = p_scene(two_blobs)
    views = []
    for v in (0, 1):
        intr, pose = p_cam(two_blobs, f"v{v}_")
        # self-consistent ground truth: this renderer's own image of the scene
        views.append(P.TrainingView(v, intr, pose, P.render(scene, intr, pose)))
    ds = P.build_edited_dataset(views, P.SelectionCloud(two_blobs["cloud"]), (1.0, 0.2, 0.2), scene)
    lines = []
    opt = P.BackgroundOptimizer(scene, ds, seed=7, metrics_sink=lambda m: lines.append(m.line()))
    final = opt.run_iterations(10)
    ref = [l.split(",") for l in two_blobs["traj_lines"]]
    got = [l.split(",") for l in lines]
    assert [g[:3] for g in got] == [r[:3] for r in ref]
    for g, r in zip(got, ref):
        for a, b in zip(g[3:], r[3:]):
            assert abs(float(a) - float(b)) < 2e-4
    assert np.abs(final.sh - two_blobs["traj_sh"]).max() < 5e-2
    np.testing.assert_array_equal(final.positions, scene.positions)


@pytest.mark.parametrize("prefetch", [0, 2])
def test_optimizer_state_resume_is_exact(two_blobs, tmp_path, prefetch):
    """save_state after 6 iterations, then 5 more == a fresh optimizer that loads
    the state and runs 5: same SH bits and the same metric lines (the views drawn
    ahead by the prefetcher are replayed before new draws)."""
    scene = p_scene(two_blobs)
    views = []
    for v in (0, 1):
        intr, pose = p_cam(two_blobs, f"v{v}_")
        views.append(P.TrainingView(v, intr, pose, P.render(scene, intr, pose)))
    ds = P.build_edited_dataset(views, P.SelectionCloud(two_blobs["cloud"]), (1.0, 0.2, 0.2), scene)
    kw = dict(seed=7, cache_views=prefetch == 0, prefetch=prefetch)
    la, lb = [], []
    a = P.BackgroundOptimizer(scene, ds, metrics_sink=lambda m: la.append(m.line()), **kw)
    a.run_iterations(6)
    a.save_state(tmp_path / "state.npz")
    sha = a.run_iterations(5).sh
    a.stop()
    b = P.BackgroundOptimizer(scene, ds, metrics_sink=lambda m: lb.append(m.line()), **kw)
    b.load_state(tmp_path / "state.npz")
    shb = b.run_iterations(5).sh
    b.stop()
    np.testing.assert_array_equal(sha, shb)
    assert lb == la[6:]


def test_self_consistent_dataset_is_fixed_point(two_blobs):
    scene = p_scene(two_blobs)
    views = []
    for v in (0, 1):
        intr, pose = p_cam(two_blobs, f"v{v}_")
        views.append(P.TrainingView(v, intr, pose, P.render(scene, intr, pose)))
    ds = P.build_edited_dataset(views, P.empty_cloud(), (1.0, 1.0, 1.0), scene)
    new_scene, state, metrics = P.optimize_iteration(scene, ds, np.random.default_rng(0),
                                                     P.AdamState.fresh(len(scene)))
    assert metrics.loss.total == 0.0
    np.testing.assert_array_equal(new_scene.sh, scene.sh)


def test_determinism(two_blobs):
    scene = p_scene(two_blobs)
    views = []
    for v in (0, 1):
        intr, pose = p_cam(two_blobs, f"v{v}_")
        views.append(P.TrainingView(v, intr, pose, P.render(scene, intr, pose)))
    ds = P.build_edited_dataset(views, P.SelectionCloud(two_blobs["cloud"]), (1.0, 0.2, 0.2), scene)
    runs = []
    for _ in range(2):
        lines = []
        opt = P.BackgroundOptimizer(scene, ds, seed=3, metrics_sink=lambda m: lines.append(m.line()))
        runs.append((opt.run_iterations(6).sh, lines))
    np.testing.assert_array_equal(runs[0][0], runs[1][0])
    assert runs[0][1] == runs[1][1]


# ---------------------------------------------------------------- larger scenes (C2 scale)
@pytest.mark.slow
def test_c2_scale_sparse_parity():
    """200k gaussians at 800x800 (config 2): kept order bit-exact vs the oracle's
    fp64 argsort; depth bit-exact and colour within 1e-4 at sampled pixels vs
    the sparse per-pixel oracle; render deterministic."""
    from paper_2511_18441_b200 import device as D
    from paper_2511_18441_b200.synthetic import ring_cameras, scaled_scene
    scene, _ = scaled_scene(200_000, 3, seed=0)
    intr, pose = ring_cameras(800, 800, 16)[5]
    view = D.View(D.device_scene(scene), intr, pose, P.DEFAULT_CONFIG)
    p = OR.project(scene, intr, pose)
    idx, z = view.kept()
    np.testing.assert_array_equal(idx.cpu().numpy(), p.index)
    img = P.render(scene, intr, pose)
    np.testing.assert_array_equal(img, P.render(scene, intr, pose))
    dep = P.depth_from_gaussians(scene, intr, pose)
    rng = np.random.default_rng(1)
    us, vs = rng.integers(0, 800, 300), rng.integers(0, 800, 300)
    col, _, odep, _ = OR.sparse_pixels(p, us, vs)
    assert np.abs(img[vs, us] - col).max() <= IMG_TOL
    np.testing.assert_array_equal(dep[vs, us], odep)


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "c1.npz")), reason="c1 golden not generated")
def test_config1_against_reference():
    """Config 1 (10k gaussians, SH deg 0, 4 views at 256^2): view-0 render and
    depth, all four selection masks, vs the reference's own outputs."""
    from conftest import load_golden
    from paper_2511_18441_b200.synthetic import ring_cameras, scaled_scene
    d = load_golden("c1.npz")
    scene, _ = scaled_scene(10_000, 0, seed=0)
    cams = ring_cameras(256, 256, 4)
    intr, pose = cams[0]
    assert_image_close(P.render(scene, intr, pose), d["v0_image"])
    assert_depth_exact(P.depth_from_gaussians(scene, intr, pose), d["v0_depth"])
    cloud = P.SelectionCloud(d["cloud"])
    for v, (intr, pose) in enumerate(cams):
        dep = P.depth_from_gaussians(scene, intr, pose)
        np.testing.assert_array_equal(P.project_cloud(cloud, intr, pose, dep), d[f"v{v}_mask"])


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "c1.npz")), reason="c1 golden not generated")
def test_config1_refit_trajectory():
    """Config 1 end to end: selection (reference cloud) + 20 refit iterations with
    seed 7.  Ground truth is each implementation's own render (self-consistent,
    SURVEY.md 8(c)(iv)); the view sequence must be identical, the per-step losses
    and the final render must track the reference run."""
    from conftest import load_golden
    from paper_2511_18441_b200.synthetic import ring_cameras, scaled_scene
    d = load_golden("c1.npz")
    scene, _ = scaled_scene(10_000, 0, seed=0)
    cams = ring_cameras(256, 256, 4)
    views = [P.TrainingView(i, intr, pose, P.render(scene, intr, pose)) for i, (intr, pose) in enumerate(cams)]
    ds = P.build_edited_dataset(views, P.SelectionCloud(d["cloud"]), (1.0, 0.2, 0.2), scene)
    for v in range(4):
        np.testing.assert_array_equal(ds.views[v].mask, d[f"v{v}_mask"])
    lines = []
    opt = P.BackgroundOptimizer(scene, ds, seed=7, metrics_sink=lambda m: lines.append(m.line()))
    final = opt.run_iterations(20)
    ref = [l.split(",") for l in d["traj_lines"]]
    got = [l.split(",") for l in lines]
    assert [g[:3] for g in got] == [r[:3] for r in ref]
    worst = max(abs(float(a) - float(b)) for g, r in zip(got, ref) for a, b in zip(g[3:], r[3:]))
    img = P.render(final, *cams[0])
    p = psnr(img, d["final_v0_render"])
    dc = np.abs(final.sh[:, 0, :] - d["traj_dc"]).max()
    print(f"c1 trajectory: worst metric diff {worst:.2e}, final render PSNR {p:.1f} dB, max |dDC| {dc:.2e}")
    assert worst < 1e-3
    assert p > 60.0  # SURVEY.md 8(c)(iv) gate


# ---------------------------------------------------------------- engine pipelines
def test_engine_pipelines_bit_identical():
    """The step pipelines are scheduling choices only: inline view builds, views
    prefetched on a side stream, and prefetching with the next view's colour
    fused into Adam (rcgs_adam_fused_next) give bit-identical SH, Adam state and
    per-step metrics."""
    import sys
    import torch
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    import bench
    from paper_2511_18441_b200.engine import RefitEngine
    cfg = dict(n=30_000, deg=3, views=6, width=320, height=240)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, torch.device("cuda", 0))
    from paper_2511_18441_b200 import device as D
    sp = P.SelectionPass(ds, cams, gt)
    sp.run(D.to_device(cloud.points, torch.float64), (1.0, 0.2, 0.2))
    targets = [sp.edited[i] for i in range(len(cams))]
    out = []
    for prefetch, fuse in ((0, False), (2, False), (2, True), (3, True)):
        eng = RefitEngine(ds, sh0.clone(), cams, targets, P.OptimizerConfig(), seed=5, cache_views=False,
                          prefetch=prefetch, fuse_color=fuse)
        for _ in range(9):
            eng.step()
        recs = [(list(map(int, p)),) + tuple(r) for p, *r in eng.drain()]
        eng.close()
        out.append((eng.sh.clone(), eng.m.clone(), eng.v.clone(), recs))
    for sh, m, v, recs in out[1:]:
        assert torch.equal(sh, out[0][0]) and torch.equal(m, out[0][1]) and torch.equal(v, out[0][2])
        assert recs == out[0][3]


def test_sparse_adam_bit_identical_to_dense():
    """Skipping the 64-gaussian tiles whose Adam state and gradient are exactly
    zero (rcgs_adam_fused_ex tile state) leaves SH, m, v and the metrics
    bit-identical to the dense update, with and without the fused colour epilogue."""
    import sys
    import torch
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    import bench
    from paper_2511_18441_b200 import device as D
    from paper_2511_18441_b200.engine import RefitEngine
    cfg = dict(n=30_000, deg=3, views=6, width=320, height=240)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, torch.device("cuda", 0))
    sp = P.SelectionPass(ds, cams, gt)
    sp.run(D.to_device(cloud.points, torch.float64), (1.0, 0.2, 0.2))
    targets = [sp.edited[i] for i in range(len(cams))]
    for prefetch in (0, 2):
        out = []
        for sparse in (False, True):
            eng = RefitEngine(ds, sh0.clone(), cams, targets, P.OptimizerConfig(), seed=5, cache_views=False,
                              prefetch=prefetch, sparse_adam=sparse)
            for _ in range(9):
                eng.step()
            recs = [repr(r) for r in eng.drain()]
            touched = None if eng.tile_state is None else float(eng.tile_state.float().mean())
            eng.close()
            out.append((eng.sh.clone(), eng.m.clone(), eng.v.clone(), recs, touched))
        assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])
        assert torch.equal(out[0][2], out[1][2]) and out[0][3] == out[1][3]
        assert 0.0 < out[1][4] <= 1.0


def test_weight_records_bit_identical():
    """rcgs_render_train + record-streaming backward + SpMV re-render equal the
    traversal render / backward bit for bit (weights depend on geometry only)."""
    import sys
    import torch
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    import bench
    from paper_2511_18441_b200 import device as D
    cfg = dict(n=40_000, deg=3, views=3, width=400, height=300)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, torch.device("cuda", 0))
    sh = sh0 + 0.01 * torch.randn_like(sh0)  # colours away from the ground truth
    for intr, pose in cams:
        ref = D.View(ds, intr, pose, P.DEFAULT_CONFIG).color(sh)
        rec = D.View(ds, intr, pose, P.DEFAULT_CONFIG).color(sh)
        img_ref, tf_ref = ref.render(None, 0, t_final=True)
        img_rec, tf_rec = rec.render(None, 0, t_final=True, train=True)
        assert torch.equal(img_ref, img_rec) and torch.equal(tf_ref, tf_rec)
        bg = np.array([0.2, 0.5, 0.9])
        assert torch.equal(ref.render(bg, 1), rec.render(bg, 1))  # SpMV path, planar layout
        g = torch.randn_like(img_ref) * 1e-3
        g[: 40] = 0.0  # zero-gradient blocks are skipped by both paths
        assert torch.equal(ref.backward(g), rec.backward(g))
        ref.close()
        rec.close()


def test_kept_records_bit_identical():
    """A view whose weights were copied into view-owned memory renders (SpMV) and
    back-propagates exactly like the traversal paths, also after another view has
    recorded into the shared arena."""
    import sys
    import torch
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    import bench
    from paper_2511_18441_b200 import device as D
    cfg = dict(n=30_000, deg=3, views=2, width=320, height=256)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, torch.device("cuda", 0))
    sh = sh0 + 0.01 * torch.randn_like(sh0)
    (i0, p0), (i1, p1) = cams
    ref = D.View(ds, i0, p0, P.DEFAULT_CONFIG).color(sh)
    kept = D.View(ds, i0, p0, P.DEFAULT_CONFIG).color(sh)
    img_ref = ref.render(None, 0)
    assert torch.equal(kept.render(None, 0, train=True), img_ref)
    kept.keep_records()
    other = D.View(ds, i1, p1, P.DEFAULT_CONFIG).color(sh)
    other.render(None, 0, train=True)  # takes over the shared arena
    assert torch.equal(kept.render(None, 0), img_ref)
    assert torch.equal(kept.render(None, 0, train=True), img_ref)
    g = torch.randn_like(img_ref) * 1e-3
    assert torch.equal(kept.backward(g), ref.backward(g))
    for v in (ref, kept, other):
        v.close()


def test_streamed_targets_pipeline_identical(two_blobs):
    """BackgroundOptimizer with host-resident targets uploaded by the prefetcher
    (copy stream) and metrics read back one step late gives the same SH and
    metric lines as the device-resident, synchronous configuration."""
    scene = p_scene(two_blobs)
    views = []
    for v in (0, 1):
        intr, pose = p_cam(two_blobs, f"v{v}_")
        views.append(P.TrainingView(v, intr, pose, P.render(scene, intr, pose)))
    ds = P.build_edited_dataset(views, P.SelectionCloud(two_blobs["cloud"]), (1.0, 0.2, 0.2), scene)
    runs = []
    for stream_targets, prefetch in ((False, 0), (True, 2)):
        lines = []
        opt = P.BackgroundOptimizer(scene, ds, seed=3, metrics_sink=lambda m: lines.append(m.line()),
                                    stream_targets=stream_targets, prefetch=prefetch)
        for _ in range(7):
            opt._step()
            opt._flush(wait=False)
        opt._flush()
        runs.append((opt._engine.sh.detach().cpu().numpy().copy(), lines))
        opt.stop()
    np.testing.assert_array_equal(runs[0][0], runs[1][0])
    assert runs[0][1] == runs[1][1]


# ---------------------------------------------------------------- select-from-mask (8(f) row 1)
def test_knn_mean_distances_bit_exact():
    """GPU kNN mean distances == scipy cKDTree + numpy mean, bit for bit, on
    uniform, surface-like (unprojected depth), duplicated and tiny clouds."""
    from scipy.spatial import cKDTree

    def ref(p, k):
        d, _ = cKDTree(p).query(p, k=k + 1)
        return d[:, 1:].mean(axis=1)

    rng = np.random.default_rng(5)
    u, v = rng.uniform(0, 1, 20000), rng.uniform(0, 1, 20000)
    surface = np.stack([u, v, 0.3 * np.sin(6 * u) + 0.01 * rng.normal(size=u.size)], axis=1)
    clouds = {
        "uniform": rng.uniform(-2, 3, (30000, 3)),
        "surface": surface,
        "dups": np.repeat(rng.uniform(0, 1, (700, 3)), 3, axis=0),
        "tiny": rng.uniform(0, 1, (18, 3)),
        "far_outliers": np.concatenate([rng.normal(size=(5000, 3)) * 0.01, rng.uniform(-50, 50, (40, 3))]),
    }
    for name, pts in clouds.items():
        for k in ((16, 5) if name != "tiny" else (16,)):
            got = P.knn_mean_distances(pts, k)
            np.testing.assert_array_equal(got, ref(pts, k), err_msg=f"{name} k={k}")
    cloud = P.SelectionCloud(clouds["far_outliers"])
    kept = P.remove_outliers(cloud, 16, 1.0)
    np.testing.assert_array_equal(kept.points, OS.remove_outliers(clouds["far_outliers"], 16, 1.0))


def test_select_from_mask_matches_reference_cloud(two_blobs):
    """unproject + GPU remove_outliers reproduce the reference's golden cloud."""
    from conftest import golden_camera
    intr, pose = golden_camera(two_blobs, "v0_")
    intr_p = P.CameraIntrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)
    pose_p = P.CameraPose(pose.rotation, pose.translation)
    mask = P.SelectionMask2D(two_blobs["brush"], intr_p, pose_p)
    cloud = P.remove_outliers(P.unproject(mask, two_blobs["v0_depth"], 0.7, 0), 16, 0.007)
    np.testing.assert_array_equal(cloud.points, two_blobs["cloud"])


# ---------------------------------------------------------------- viewer frames (8(f) row 2)
def test_render_rgba_bit_identical_to_host_frame():
    """rcgs_render_rgba == image_to_rgba(overlay(render)) computed on the host
    (session.py:381-405), with and without a selection, for the traversal and
    the recorded-weights (SpMV) render paths."""
    import sys
    import torch
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    import bench
    from paper_2511_18441_b200 import device as D
    cfg = dict(n=30_000, deg=3, views=1, width=320, height=240)
    scene, cams, ds, sh0, gt, cloud, _ = bench.build_workload(cfg, 0, torch.device("cuda", 0))
    intr, pose = cams[0]
    v = D.View(ds, intr, pose, P.DEFAULT_CONFIG).color(sh0 * 1.7)  # some values beyond 1 (clipped)
    img = v.render(None, 0).double().cpu().numpy()
    bits = np.random.default_rng(3).uniform(size=(intr.height, intr.width)) < 0.3
    bits_dev = torch.from_numpy(bits.astype(np.uint8)).cuda()
    for train in (False, True):
        if train:
            v.render(None, 0, train=True)  # later renders stream the recorded weights
        np.testing.assert_array_equal(v.render_rgba().cpu().numpy(), P.image_to_rgba(img))
        np.testing.assert_array_equal(v.render_rgba(bits_dev).cpu().numpy(),
                                      P.image_to_rgba(P.overlay(img, bits)))
    v.close()


_LAYOUT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2511_18441_b200 as P
from paper_2511_18441_b200.synthetic import ring_cameras, scaled_scene
scene, _ = scaled_scene(60_000, 3, seed=4)
out = []
for intr, pose in ring_cameras(640, 360, 3):
    out.append(P.render(scene, intr, pose))
    out.append(P.depth_from_gaussians(scene, intr, pose))
    cap = P.render_forward(scene, intr, pose)
    out.append(P.backward_sh(cap, np.full((360, 640, 3), 1e-3) * (np.arange(640) % 7 - 3)[None, :, None]))
np.savez(sys.argv[2], *out)
"""


def test_tile_list_layouts_agree(tmp_path):
    """The pair-mask layouts: masks packed above the scene index (scenes below 2^24
    gaussians) and the large-scene layout (plain indices + a mask array, forced
    with RCGS_PAIR_PACK=0) give bit-identical render, depth and backward."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "layout.py"
    script.write_text(_LAYOUT_SCRIPT)
    res = {}
    for pack in ("1", "0"):
        out = tmp_path / f"o{pack}.npz"
        env = dict(os.environ, RCGS_PAIR_PACK=pack)
        subprocess.run([sys.executable, str(script), root, str(out)], check=True, env=env, timeout=600)
        res[pack] = np.load(out)
    for key in res["1"].files:
        np.testing.assert_array_equal(res["1"][key], res["0"][key])


@pytest.mark.gpu
def test_color_activation_boundary_exact():
    """The per-step colour is evaluated in fp32 with an fp64 fallback for the
    activation decision raw + 0.5 > 0 (render.py:211-214): gaussians whose DC
    coefficient puts raw + 0.5 within a few fp32 ulps of 0 must get the fp64
    reference's decision, both from color_kernel and from the Adam colour
    epilogue (which must also agree with color_kernel bit for bit)."""
    import ctypes
    import torch
    from paper_2511_18441_b200 import _native as N, device as D
    from oracle.raster import sh_basis, camera_center
    rng = np.random.default_rng(5)
    n = 4000
    pos = np.column_stack([rng.uniform(-1.2, 1.2, n), rng.uniform(-0.9, 0.9, n), rng.uniform(2.0, 4.0, n)])
    rot = rng.normal(size=(n, 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    scl = rng.uniform(0.005, 0.03, (n, 3))
    opa = rng.uniform(0.3, 0.9, n)
    sh = (rng.normal(size=(n, 16, 3)) * 0.05).astype(np.float32).astype(np.float64)
    intr = P.CameraIntrinsics(300.0, 300.0, 159.5, 119.5, 320, 240)
    pose = P.CameraPose(np.eye(3), np.zeros(3))
    d = pos - camera_center(pose)
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    basis = sh_basis(d, 3)
    rest = np.einsum("nk,nkc->nc", basis[:, 1:], sh[:, 1:])
    c0 = ((-0.5 - rest) / basis[:, :1]).astype(np.float32)  # raw + 0.5 ~ 0 in every channel
    nudge = rng.integers(-3, 4, size=(n, 3))
    for k in range(1, 4):  # move some channels by k fp32 ulps either way
        c0 = np.where(nudge >= k, np.nextafter(c0, np.float32(np.inf)), c0)
        c0 = np.where(nudge <= -k, np.nextafter(c0, np.float32(-np.inf)), c0)
    sh[:, 0, :] = c0.astype(np.float64)
    scene = P.Scene(pos, rot, scl, opa, sh, 3)
    ref = OR.project(scene, intr, pose)
    raw64 = np.einsum("nk,nkc->nc", ref.basis, sh[ref.index]) + 0.5
    assert np.mean(np.abs(raw64) < 1e-5) > 0.9  # the fp32 band is exercised
    clear = np.abs(raw64) > 1e-13                 # decisions independent of the fp64 sum order
    cap = P.render_forward(scene, intr, pose)
    np.testing.assert_array_equal(cap.kept_index, ref.index)
    assert np.array_equal(cap.active[clear], ref.active[clear])

    # the fused colour epilogue of a zero-gradient Adam step (SH unchanged) on the same view
    ds = D.DeviceScene(scene.positions, scene.rotations, scene.scales, scene.opacities, 3)
    sh_dev = torch.from_numpy(sh.astype(np.float32)).cuda().contiguous()
    v_ref = D.View(ds, intr, pose, P.DEFAULT_CONFIG).color(sh_dev)
    v_fused = D.View(ds, intr, pose, P.DEFAULT_CONFIG)
    m = torch.zeros_like(sh_dev)
    v = torch.zeros_like(sh_dev)
    acc = torch.zeros((n, 3), dtype=torch.float32, device="cuda")
    reject = torch.zeros(1, dtype=torch.int32, device="cuda")
    step = torch.zeros(1, dtype=torch.int64, device="cuda")
    rec = torch.zeros(1, dtype=torch.float64, device="cuda")
    cfg = D.adam_config(P.OptimizerConfig())
    ptrs = (ctypes.c_void_p * 1)(acc.data_ptr())
    cen = (ctypes.c_double * 3)(*camera_center(pose))
    sh_before = sh_dev.clone()
    N.call("rcgs_adam_fused_next", ds.handle, N.ptr(sh_dev), N.ptr(m), N.ptr(v), ptrs, cen, 1, ctypes.byref(cfg),
           N.ptr(reject), N.ptr(step), N.ptr(rec), v_fused.handle, D.stream_ptr())
    v_fused._colored = True
    assert torch.equal(sh_dev, sh_before)
    assert torch.equal(v_fused.render(None, 0), v_ref.render(None, 0))
    k = v_ref.n_kept
    outs = []
    for view in (v_ref, v_fused):
        b = torch.empty((k, 16), dtype=torch.float64, device="cuda")
        a = torch.empty((k, 3), dtype=torch.uint8, device="cuda")
        N.call("rcgs_view_basis", view.handle, N.ptr(b), N.ptr(a), D.stream_ptr())
        outs.append(a.cpu().numpy().astype(bool))
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[1][clear], ref.active[clear])
    v_ref.close()
    v_fused.close()
