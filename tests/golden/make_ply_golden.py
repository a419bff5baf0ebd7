"""Golden PLY checkpoints from the REAL reference (`splattint.scene_io`), for
SURVEY.md 8(f) row 4.  Run once in the build container (the only place
/root/reference exists); the outputs travel with the repo.

    python tests/golden/make_ply_golden.py

Outputs (tests/golden/):
  ply_saved.ply      reference save_scene_ply of the scene in ply_golden.npz[src_*]
                     (saturated opacities exercise the logit clamp)
  ply_mixed.ply      hand-built: shuffled property order, extra float/uchar
                     properties, an empty `face` element, unnormalised quaternions
  ply_double.ply     as ply_mixed but with some float64 / int16 properties
  ply_golden.npz     reference load_scene_ply of each file above (<name>_<field>)
  ply_bad/*.ply      malformed / invalid files; ply_errors.json has the reference's
                     exception class and message for each
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from splattint import scene_io as ref  # noqa: E402
from splattint.scene import Scene  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
REQ = ref._REQUIRED_PROPERTIES


def source_scene(n=257, seed=3):
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    opa = rng.uniform(0.01, 0.99, n)
    opa[:4] = [1e-9, 1 - 1e-9, 1e-6, 0.999999]  # beyond / at the logit clamp
    return Scene(positions=rng.normal(size=(n, 3)) * 2.0, rotations=q, scales=np.exp(rng.normal(-3, 1, (n, 3))),
                 opacities=opa, sh=rng.normal(size=(n, 16, 3)) * 0.4)


def write_ply(path, fields, rows, extra_elements=("face 0",)):
    lines = ["ply", "format binary_little_endian 1.0", "comment made by make_ply_golden.py",
             f"element vertex {len(rows)}"]
    lines += [f"property {t} {name}" for name, t in fields]
    for e in extra_elements:
        lines += [f"element {e}", "property list uchar int vertex_indices"]
    lines.append("end_header")
    with open(path, "wb") as fh:
        fh.write(("\n".join(lines) + "\n").encode("ascii"))
        fh.write(rows.tobytes())


NP = {"float": "<f4", "double": "<f8", "uchar": "u1", "short": "<i2"}


def mixed_rows(n, seed, types):
    rng = np.random.default_rng(seed)
    names = list(REQ) + ["nx", "ny", "nz", "flags"]
    order = rng.permutation(len(names))
    fields = [(names[i], types.get(names[i], "uchar" if names[i] == "flags" else "float")) for i in order]
    rows = np.zeros(n, dtype=np.dtype([(k, NP[t]) for k, t in fields]))
    for k, t in fields:
        if t == "uchar":
            rows[k] = rng.integers(0, 255, n)
        elif t == "short":
            rows[k] = rng.integers(-5, 5, n)
        else:
            rows[k] = rng.normal(size=n) * (0.5 if k.startswith("f_") else 1.5)
    for i in range(4):
        rows[f"rot_{i}"] = rng.normal(size=n) * 3.0  # unnormalised
    return fields, rows


def main():
    os.makedirs(os.path.join(OUT, "ply_bad"), exist_ok=True)
    out = {}
    src = source_scene()
    for f in ("positions", "rotations", "scales", "opacities", "sh"):
        out[f"src_{f}"] = getattr(src, f)
    ref.save_scene_ply(src, os.path.join(OUT, "ply_saved.ply"))
    fields, rows = mixed_rows(131, 5, {})
    write_ply(os.path.join(OUT, "ply_mixed.ply"), fields, rows)
    fields, rows = mixed_rows(67, 6, {"x": "double", "opacity": "double", "f_rest_7": "double", "scale_1": "short"})
    write_ply(os.path.join(OUT, "ply_double.ply"), fields, rows, ())
    for name in ("saved", "mixed", "double"):
        sc = ref.load_scene_ply(os.path.join(OUT, f"ply_{name}.ply"))
        for f in ("positions", "rotations", "scales", "opacities", "sh"):
            out[f"{name}_{f}"] = getattr(sc, f)
    np.savez_compressed(os.path.join(OUT, "ply_golden.npz"), **out)

    # invalid files: (name, header lines, row-dtype fields, row mutator, payload cut)
    bad = {}
    base_fields = [(k, "float") for k in REQ]

    def good_rows(n=9):
        rng = np.random.default_rng(11)
        rows = np.zeros(n, dtype=np.dtype([(k, "<f4") for k in REQ]))
        for k in REQ:
            rows[k] = rng.normal(size=n)
        return rows

    def emit(name, text_lines, payload):
        path = os.path.join(OUT, "ply_bad", f"{name}.ply")
        with open(path, "wb") as fh:
            fh.write(("\n".join(text_lines) + "\n").encode("ascii"))
            fh.write(payload)
        try:
            ref.load_scene_ply(path)
            bad[name] = None
        except Exception as exc:  # noqa: BLE001 - recording the reference's behaviour
            bad[name] = [type(exc).__name__, str(exc)]

    def header(n, fields=base_fields, fmt="binary_little_endian", extra=()):
        h = ["ply", f"format {fmt} 1.0", f"element vertex {n}"] + [f"property {t} {k}" for k, t in fields]
        return h + list(extra) + ["end_header"]

    rows = good_rows()
    for grp, col in (("position", "y"), ("opacity", "opacity"), ("scale", "scale_2"), ("rotation", "rot_1"),
                     ("f_dc", "f_dc_0"), ("f_rest", "f_rest_44")):
        r = rows.copy()
        r[col][5] = np.nan if grp != "scale" else np.inf
        r["x"][7] = np.inf if grp == "f_rest" else r["x"][7]  # an earlier group failing later
        emit(f"nonfinite_{grp}", header(len(r)), r.tobytes())
    r = rows.copy()
    for i in range(4):
        r[f"rot_{i}"][3] = 0.0
    emit("zero_quaternion", header(len(r)), r.tobytes())
    emit("truncated", header(len(rows)), rows.tobytes()[:-3])
    emit("missing_property", header(len(rows), [f for f in base_fields if f[0] != "f_rest_17"]), b"")
    emit("ascii_format", header(len(rows), fmt="ascii"), rows.tobytes())
    emit("not_ply", ["plyx"], b"")
    emit("list_in_vertex", header(0, base_fields + [("idx", "list uchar int")]), b"")
    emit("unknown_type", header(0, base_fields + [("h", "half")]), b"")
    emit("nonempty_face", header(len(rows), extra=["element face 2", "property list uchar int vertex_indices"]),
         rows.tobytes())
    emit("no_vertex", ["ply", "format binary_little_endian 1.0", "element face 0", "end_header"], b"")
    emit("unterminated", ["ply", "format binary_little_endian 1.0", "element vertex 0"][:3], b"")
    emit("empty_ok", header(0), b"")
    with open(os.path.join(OUT, "ply_errors.json"), "w") as fh:
        json.dump(bad, fh, indent=1, sort_keys=True)
    print(json.dumps(bad, indent=1))


if __name__ == "__main__":
    main()
