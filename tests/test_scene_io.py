"""PLY checkpoints (reference scene_io.py:108-180,
tests test_scene_io.py:49-170).  Host functions against the golden files made by
the reference (tests/golden/make_ply_golden.py); the GPU decode / encode against
the host functions, bit for bit."""

from __future__ import annotations

import json
import os
import struct

import numpy as np
import pytest

import paper_2511_18441_b200 as P
from paper_2511_18441_b200 import errors
from paper_2511_18441_b200 import scene_io as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FIELDS = ("positions", "rotations", "scales", "opacities", "sh")


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLD, "ply_golden.npz"))


def _src_scene(g):
    return P.Scene(*(g[f"src_{f}"] for f in FIELDS))


def _bad_cases():
    with open(os.path.join(GOLD, "ply_errors.json")) as fh:
        return sorted(json.load(fh).items())


def _raw_row(position=(0.0, 0.0, 0.0), f_dc=(0.0, 0.0, 0.0), f_rest=None, opacity=0.0, scale=(0.0, 0.0, 0.0),
             rot=(1.0, 0.0, 0.0, 0.0)):
    rest = [0.0] * 45 if f_rest is None else list(f_rest)
    return list(position) + list(f_dc) + rest + [opacity] + list(scale) + list(rot)


def _write_raw(path, rows):
    head = ["ply", "format binary_little_endian 1.0", f"element vertex {len(rows)}"]
    head += [f"property float {k}" for k in S.PROPERTY_ORDER] + ["end_header"]
    with open(path, "wb") as fh:
        fh.write(("\n".join(head) + "\n").encode("ascii"))
        for r in rows:
            fh.write(struct.pack(f"<{len(r)}f", *r))


@pytest.mark.parametrize("name", ["saved", "mixed", "double"])
def test_load_matches_reference(golden, name):
    sc = P.load_scene_ply(os.path.join(GOLD, f"ply_{name}.ply"))
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(sc, f), golden[f"{name}_{f}"], err_msg=f)


def test_save_byte_identical_to_reference(golden, tmp_path):
    out = tmp_path / "s.ply"
    P.save_scene_ply(_src_scene(golden), out)
    with open(os.path.join(GOLD, "ply_saved.ply"), "rb") as fh:
        assert out.read_bytes() == fh.read()


@pytest.mark.parametrize("case,expect", _bad_cases())
def test_errors_match_reference(case, expect):
    path = os.path.join(GOLD, "ply_bad", f"{case}.ply")
    if expect is None:
        assert len(P.load_scene_ply(path)) == 0
        return
    with pytest.raises(getattr(errors, expect[0])) as ei:
        P.load_scene_ply(path)
    assert str(ei.value) == expect[1]


def test_identity_stored_values(tmp_path):
    """test_scene_io.py:50-69: exp(0)=1, sigmoid(0)=0.5, renormalised quaternion, channel-major f_rest."""
    rest = [0.01 * (i + 1) for i in range(45)]
    _write_raw(tmp_path / "one.ply", [_raw_row((1.0, 2.0, 3.0), (0.5, 0.25, -0.125), rest, rot=(2.0, 0, 0, 0))])
    sc = P.load_scene_ply(tmp_path / "one.ply")
    np.testing.assert_array_equal(sc.positions[0], [1.0, 2.0, 3.0])
    np.testing.assert_array_equal(sc.scales[0], [1.0, 1.0, 1.0])
    assert sc.opacities[0] == 0.5
    np.testing.assert_array_equal(sc.rotations[0], [1.0, 0.0, 0.0, 0.0])
    for c in range(3):
        np.testing.assert_array_equal(sc.sh[0, 1:, c], np.float32(rest[15 * c:15 * (c + 1)]))


def test_second_roundtrip_exact(golden, tmp_path):
    """test_scene_io.py:143-166: after one float32 quantisation save/load is the identity."""
    P.save_scene_ply(_src_scene(golden), tmp_path / "a.ply")
    once = P.load_scene_ply(tmp_path / "a.ply")
    P.save_scene_ply(once, tmp_path / "b.ply")
    twice = P.load_scene_ply(tmp_path / "b.ply")
    for f in ("positions", "scales", "sh"):
        np.testing.assert_array_equal(getattr(once, f), getattr(twice, f))
    np.testing.assert_allclose(twice.opacities, once.opacities, atol=1e-6)
    np.testing.assert_allclose(twice.rotations, once.rotations, atol=1e-6)


def test_empty_scene_roundtrip(tmp_path):
    sc = P.Scene(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 16, 3)))
    P.save_scene_ply(sc, tmp_path / "e.ply")
    assert len(P.load_scene_ply(tmp_path / "e.ply")) == 0


# --------------------------------------------------------------------------- GPU
def _device_geometry(ds):
    return {"positions": ds.positions.cpu().numpy(), "rotations": ds.rotations.cpu().numpy(),
            "scales": ds.scales.cpu().numpy(), "opacities": ds.opacities.cpu().numpy()}


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["saved", "mixed", "double"])
def test_device_load_bit_identical(golden, name):
    ds, sh = P.load_scene_ply_device(os.path.join(GOLD, f"ply_{name}.ply"))
    got = _device_geometry(ds)
    for f in ("positions", "rotations", "scales", "opacities"):
        np.testing.assert_array_equal(got[f], golden[f"{name}_{f}"], err_msg=f)
    np.testing.assert_array_equal(sh.cpu().numpy(), golden[f"{name}_sh"].astype(np.float32))
    ds.close()


@pytest.mark.gpu
@pytest.mark.parametrize("case,expect", _bad_cases())
def test_device_load_errors_match_reference(case, expect):
    path = os.path.join(GOLD, "ply_bad", f"{case}.ply")
    if expect is None:
        ds, sh = P.load_scene_ply_device(path)
        assert ds.n == 0 and tuple(sh.shape) == (0, 16, 3)
        return
    with pytest.raises(getattr(errors, expect[0])) as ei:
        P.load_scene_ply_device(path)
    assert str(ei.value) == expect[1]


@pytest.mark.gpu
def test_device_save_byte_identical(golden, tmp_path):
    import torch

    from paper_2511_18441_b200 import device as D
    from paper_2511_18441_b200.optimize import _delta_to_host

    scene = _src_scene(golden)
    old = D.sh_to_device(scene.sh)
    g = torch.Generator(device="cuda").manual_seed(0)
    new = old + 1e-3 * torch.randn(old.shape, device="cuda", generator=g)
    new[::3] = old[::3]  # untouched rows keep the host fp64 value
    base = torch.from_numpy(scene.sh).cuda()
    S.save_scene_ply_device(scene, new, tmp_path / "d.ply", sh_base=(base, old))
    P.save_scene_ply(scene.with_sh(_delta_to_host(scene.sh, old, new)), tmp_path / "h.ply")
    assert (tmp_path / "d.ply").read_bytes() == (tmp_path / "h.ply").read_bytes()
    S.save_scene_ply_device(scene, new, tmp_path / "d2.ply")
    P.save_scene_ply(scene.with_sh(new.double().cpu().numpy()), tmp_path / "h2.ply")
    assert (tmp_path / "d2.ply").read_bytes() == (tmp_path / "h2.ply").read_bytes()


@pytest.mark.gpu
def test_optimizer_save_matches_current_scene(two_blobs, tmp_path):
    """criterion 8 (bit-identical PLY): the device save of a running refit equals
    save_scene_ply(current_scene()) byte for byte."""
    from test_gpu_parity import p_cam, p_scene

    scene = p_scene(two_blobs)
    views = []
    for v in (0, 1):
        intr, pose = p_cam(two_blobs, f"v{v}_")
        views.append(P.TrainingView(v, intr, pose, P.render(scene, intr, pose)))
    ds = P.build_edited_dataset(views, P.SelectionCloud(two_blobs["cloud"]), (1.0, 0.2, 0.2), scene)
    opt = P.BackgroundOptimizer(scene, ds, seed=7)
    opt.run_iterations(5)
    opt.save_ply(tmp_path / "d.ply")
    P.save_scene_ply(opt.current_scene(), tmp_path / "h.ply")
    assert (tmp_path / "d.ply").read_bytes() == (tmp_path / "h.ply").read_bytes()
