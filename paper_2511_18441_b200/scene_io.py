"""3DGS PLY checkpoints (scene_io.py:108-180).

Layout (the reference's): binary little-endian, one non-empty `vertex` element,
properties x y z, f_dc_0..2, f_rest_0..44 (channel-major: 15 red, 15 green,
15 blue), opacity (logit), scale_0..2 (log), rot_0..3 (w x y z, unnormalised);
extra vertex properties are ignored on load.

Host functions (`load_scene_ply`, `save_scene_ply`) keep the reference's values
and errors.  The device functions move the per-gaussian work of a checkpoint to
the GPU around the optimizer's state:

* `load_scene_ply_device` uploads the float32 rows once and decodes them with
  rcgs_ply_decode into the DeviceScene's fp64 positions / normalised rotations
  and the optimizer's (N, 16, 3) fp32 SH; only exp / sigmoid of the 4
  transcendental columns run in numpy, so every value equals the host loader's.
* `save_scene_ply_device` writes the SH columns of a device-resident row buffer
  (geometry columns encoded once per scene, cached) with rcgs_ply_encode_sh and
  reads it back in one D2H copy: the file is byte-identical to
  `save_scene_ply` of the published snapshot (optimize.py:226-238).
"""

from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict

import numpy as np
import torch

from . import _native as N
from . import device as D
from .errors import DataError, FormatError
from .scene import Scene

SH_REST = 45
OPACITY_LOGIT_CLAMP = 13.9  # scene_io.py:34 (sigmoid(13.9) is 1 - 9.2e-7)
PROPERTY_ORDER = (("x", "y", "z") + tuple(f"f_dc_{i}" for i in range(3))
                  + tuple(f"f_rest_{i}" for i in range(SH_REST)) + ("opacity",)
                  + tuple(f"scale_{i}" for i in range(3)) + tuple(f"rot_{i}" for i in range(4)))
# column order shared with rcgs_ply_decode / rcgs_ply_encode_sh
DECODE_ORDER = (("x", "y", "z") + tuple(f"rot_{i}" for i in range(4)) + tuple(f"f_dc_{i}" for i in range(3))
                + tuple(f"f_rest_{i}" for i in range(SH_REST)) + ("opacity",) + tuple(f"scale_{i}" for i in range(3)))
_POS, _ROT, _DC, _REST, _OPA, _SCL = slice(0, 3), slice(3, 7), slice(7, 10), slice(10, 55), 55, slice(56, 59)

_SCALAR_TYPES = {}
for _names, _code in ((("float", "float32"), "<f4"), (("double", "float64"), "<f8"), (("uchar", "uint8"), "u1"),
                      (("char", "int8"), "i1"), (("short", "int16"), "<i2"), (("ushort", "uint16"), "<u2"),
                      (("int", "int32"), "<i4"), (("uint", "uint32"), "<u4")):
    for _n in _names:
        _SCALAR_TYPES[_n] = _code


class PlyLayout:
    """Parsed header: vertex count, the row dtype and where the payload starts."""

    def __init__(self, count: int, dtype: np.dtype, data_offset: int):
        self.count, self.dtype, self.data_offset = count, dtype, data_offset

    @property
    def all_float32(self) -> bool:
        return all(self.dtype[name] == np.dtype("<f4") for name in self.dtype.names)

    def float_offsets(self):
        """ctypes int32[59] of DECODE_ORDER's positions, in floats, within a row."""
        return (ctypes.c_int32 * len(DECODE_ORDER))(*[self.dtype.fields[k][1] // 4 for k in DECODE_ORDER])


def read_ply_layout(fh) -> PlyLayout:
    """Header grammar and errors of scene_io.py:63-105 (+ the required-property check, 112-114)."""
    if fh.readline().strip() != b"ply":
        raise FormatError("not a PLY file")
    state = {"format": None, "element": None}
    elements, fields = [], []

    def on_format(tok):
        state["format"] = tok[1]

    def on_element(tok):
        state["element"] = tok[1]
        elements.append((tok[1], int(tok[2])))

    def on_property(tok):
        if state["element"] != "vertex":
            return
        if tok[1] == "list":
            raise FormatError("list properties not supported in vertex element")
        code = _SCALAR_TYPES.get(tok[1])
        if code is None:
            raise FormatError(f"unsupported property type {tok[1]!r}")
        fields.append((tok[2], code))

    handlers = {"format": on_format, "element": on_element, "property": on_property}
    while True:
        raw = fh.readline()
        if not raw:
            raise FormatError("unterminated PLY header")
        tok = raw.decode("ascii", errors="replace").split()
        if not tok or tok[0] == "comment":
            continue
        if tok[0] == "end_header":
            break
        if tok[0] in handlers:
            handlers[tok[0]](tok)
    if state["format"] != "binary_little_endian":
        raise FormatError(f"unsupported PLY format {state['format']!r} (need binary_little_endian)")
    counts = [c for name, c in elements if name == "vertex"]
    if not counts:
        raise FormatError("PLY has no vertex element")
    for name, c in elements:
        if name != "vertex" and c != 0:
            raise FormatError(f"unsupported non-empty element {name!r}")
    present = {name for name, _ in fields}
    for name in PROPERTY_ORDER:
        if name not in present:
            raise FormatError(f"missing PLY property {name!r}")
    return PlyLayout(counts[0], np.dtype(fields), fh.tell())


def _read(path):
    with open(path, "rb") as fh:
        layout = read_ply_layout(fh)
        size = layout.count * layout.dtype.itemsize
        payload = fh.read(size)
    if len(payload) != size:
        raise FormatError("truncated PLY payload")
    return layout, payload


def _raise_first_bad(bad):
    """bad[k] = first offending vertex or -1, k over (position, opacity, scale,
    rotation, f_dc, f_rest, zero-norm quaternion) -- the reference's check order."""
    for k, what in enumerate(("position", "opacity", "scale", "rotation", "f_dc", "f_rest")):
        if bad[k] >= 0:
            raise DataError(f"non-finite {what} at vertex {int(bad[k])}")
    if bad[6] >= 0:
        raise DataError(f"zero-norm quaternion at vertex {int(bad[6])}")


def _activate(rows):
    """exp(log-scale), sigmoid(logit) (scene_io.py:148-150), evaluated on contiguous
    (n, 3) / (n,) float64 arrays like the reference's, so numpy takes the same loops."""
    raw_scales = np.stack([rows[f"scale_{i}"].astype(np.float64) for i in range(3)], axis=1)
    raw_opacity = np.ascontiguousarray(rows["opacity"], dtype=np.float64)
    return np.exp(raw_scales), 1.0 / (1.0 + np.exp(-raw_opacity))


def load_scene_ply(path) -> Scene:
    """Host loader (scene_io.py:108-153)."""
    layout, payload = _read(path)
    rows = np.frombuffer(payload, dtype=layout.dtype)
    n = layout.count
    cols = np.empty((n, len(DECODE_ORDER)))
    for k, name in enumerate(DECODE_ORDER):
        cols[:, k] = rows[name]
    bad = [-1] * 7
    if n:
        for k, grp in enumerate((_POS, _OPA, _SCL, _ROT, _DC, _REST)):
            hit = np.flatnonzero(~np.isfinite(cols[:, grp]).reshape(n, -1).all(axis=1))
            bad[k] = int(hit[0]) if hit.size else -1
        _raise_first_bad(bad)
    quat = cols[:, _ROT]
    norms = np.linalg.norm(quat, axis=1)
    if np.any(norms < 1e-12):
        raise DataError(f"zero-norm quaternion at vertex {int(np.argmin(norms))}")
    sh = np.empty((n, 16, 3))
    sh[:, 0, :] = cols[:, _DC]
    sh[:, 1:, :] = np.swapaxes(cols[:, _REST].reshape(n, 3, 15), 1, 2)
    scales, opacities = _activate(rows)
    return Scene(positions=cols[:, _POS], rotations=quat / norms[:, None], scales=scales, opacities=opacities,
                 sh=sh)


def _header_bytes(n: int) -> bytes:
    lines = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
    lines += [f"property float {name}" for name in PROPERTY_ORDER]
    return ("\n".join(lines + ["end_header"]) + "\n").encode("ascii")


_ROW_DTYPE = np.dtype([(name, "<f4") for name in PROPERTY_ORDER])


def _geometry_rows(scene) -> np.ndarray:
    """Rows with every non-SH column encoded (scene_io.py:167-172); SH columns zero."""
    rows = np.zeros(len(scene), dtype=_ROW_DTYPE)
    for i, axis in enumerate("xyz"):
        rows[axis] = scene.positions[:, i]
    lo, hi = 1.0 / (1.0 + np.exp(OPACITY_LOGIT_CLAMP)), 1.0 / (1.0 + np.exp(-OPACITY_LOGIT_CLAMP))
    p = np.clip(scene.opacities, lo, hi)
    rows["opacity"] = np.log(p / (1.0 - p))
    for i in range(3):
        rows[f"scale_{i}"] = np.log(scene.scales[:, i])
    for i in range(4):
        rows[f"rot_{i}"] = scene.rotations[:, i]
    return rows


def save_scene_ply(scene: Scene, path) -> None:
    """Host writer (scene_io.py:156-180): float32 payload, clamped logit opacities."""
    n = len(scene)
    rows = _geometry_rows(scene)
    channel_major = np.swapaxes(scene.sh[:, 1:, :], 1, 2).reshape(n, SH_REST)
    for c in range(3):
        rows[f"f_dc_{c}"] = scene.sh[:, 0, c]
    for k in range(SH_REST):
        rows[f"f_rest_{k}"] = channel_major[:, k]
    with open(path, "wb") as fh:
        fh.write(_header_bytes(n))
        fh.write(rows.tobytes())


def load_scene_ply_device(path, sh_degree: int = 3):
    """(DeviceScene, (N, 16, 3) fp32 SH on the device) from a checkpoint.

    Equal to (DeviceScene.from_scene(s), sh_to_device(s.sh)) for s = load_scene_ply(path),
    with the same errors; rows with non-float32 properties take that host path."""
    with open(path, "rb") as fh:
        layout = read_ply_layout(fh)
        n = layout.count
        fast = n > 0 and layout.all_float32
        if fast:  # the payload goes straight into pinned memory
            host = torch.empty((n, layout.dtype.itemsize // 4), dtype=torch.float32, pin_memory=True)
            got = fh.readinto(memoryview(host.numpy()).cast("B"))
            if got != n * layout.dtype.itemsize:
                raise FormatError("truncated PLY payload")
    if not fast:
        scene = load_scene_ply(path)
        return D.DeviceScene.from_device(
            *(torch.from_numpy(np.ascontiguousarray(a)).to(D.device())
              for a in (scene.positions, scene.rotations, scene.scales, scene.opacities)),
            sh_degree), D.sh_to_device(scene.sh)
    dev = D.device()
    row_floats = host.shape[1]
    d_rows = host.to(dev, non_blocking=True)
    pos = torch.empty((n, 3), dtype=torch.float64, device=dev)
    rot = torch.empty((n, 4), dtype=torch.float64, device=dev)
    sh = torch.empty((n, 16, 3), dtype=torch.float32, device=dev)
    bad = (ctypes.c_int64 * 7)()
    N.call("rcgs_ply_decode", N.ptr(d_rows), n, row_floats, layout.float_offsets(), N.ptr(pos), N.ptr(rot),
           N.ptr(sh), bad, D.stream_ptr())
    _raise_first_bad(list(bad))
    scales, opacities = _activate(host.numpy().view(layout.dtype).reshape(n))
    ds = D.DeviceScene.from_device(pos, rot, torch.from_numpy(scales).to(dev),
                                   torch.from_numpy(opacities).to(dev), sh_degree)
    return ds, sh


class _GeometryCache:
    """Device copies of a scene's geometry rows, keyed on the geometry arrays."""

    def __init__(self, size: int = 2):
        self._lock = threading.Lock()
        self._items: "OrderedDict[tuple, tuple]" = OrderedDict()
        self._size = size

    def get(self, scene) -> torch.Tensor:
        key = (id(scene.positions), id(scene.rotations), id(scene.scales), id(scene.opacities),
               torch.cuda.current_device())
        with self._lock:
            hit = self._items.get(key)
            if hit is not None:
                self._items.move_to_end(key)
                return hit[1]
        rows = _geometry_rows(scene)
        dev_rows = torch.from_numpy(rows.view(np.float32).reshape(len(scene), -1)).to(D.device())
        with self._lock:
            self._items[key] = ((scene.positions, scene.rotations, scene.scales, scene.opacities), dev_rows)
            while len(self._items) > self._size:
                self._items.popitem(last=False)
        return dev_rows


_geometry_cache = _GeometryCache()
_STD_OFFSETS = PlyLayout(0, _ROW_DTYPE, 0).float_offsets()


def encode_scene_rows(scene, sh_dev: torch.Tensor, sh_base=None) -> torch.Tensor:
    """(N, 62) float32 device rows of `scene` with SH from the device.

    sh_base = (fp64 host-value SH on the device, the fp32 device SH it was taken at)
    publishes float32(base + (sh_dev - old)), the value `snapshot()` hands out."""
    n = len(scene)
    if tuple(sh_dev.shape) != (n, 16, 3) or sh_dev.dtype != torch.float32:
        raise ValueError(f"sh_dev must be ({n}, 16, 3) float32, got {tuple(sh_dev.shape)} {sh_dev.dtype}")
    rows = _geometry_cache.get(scene).clone()
    base, old = (None, None) if sh_base is None else sh_base
    N.call("rcgs_ply_encode_sh", N.ptr(base) if base is not None else None,
           N.ptr(old) if old is not None else None, N.ptr(sh_dev.contiguous()), n, rows.shape[1], _STD_OFFSETS,
           N.ptr(rows), D.stream_ptr())
    return rows


def save_scene_ply_device(scene, sh_dev: torch.Tensor, path, sh_base=None) -> None:
    """Write `scene` with device SH; byte-identical to save_scene_ply(scene.with_sh(...))."""
    rows = encode_scene_rows(scene, sh_dev, sh_base)
    host = torch.empty(rows.shape, dtype=torch.float32, pin_memory=True)
    host.copy_(rows, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    with open(path, "wb") as fh:
        fh.write(_header_bytes(len(scene)))
        fh.write(memoryview(host.numpy()).cast("B"))
