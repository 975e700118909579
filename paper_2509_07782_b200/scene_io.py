"""Scene / camera file ingestion (the file formats of the reference's
scene_io.py).

* `.gsx` records: `scene.save_scene` / `scene.load_scene` (bit-exact).
* Cameras JSON (schema of scene_io.py:114-155): a table-driven codec
  (`_CAMERA_SCHEMA`) -- one entry per JSON key with its Camera attribute,
  converter and default -- used by both `save_cameras` and `load_cameras`.
* 3DGS PLY (scene_io.py:287-380): `read_ply_vertices` parses the header into
  an element table, then decodes the vertex block in one shot (a structured
  numpy dtype for binary little-endian, `np.loadtxt` over the vertex lines for
  ascii).  `ply_records` converts all rows at once to the 87-float record
  layout exactly as the reference's GaussianShape / AppearanceCoeffs
  ingestion does (quaternion normalized in float64, scales exp'd and clamped
  at S_MIN, sigma~ = -ln(1 - alpha)/dt_ref with alpha = clip(sigmoid(opacity),
  1e-6, 1 - 1e-6), SH DC from f_dc, lobes of `AppearanceCoeffs.constant`) and
  hands the [N,87] float32 block to the device in one copy
  (`Scene.from_records`).
"""

from __future__ import annotations

import io
import json
from pathlib import Path

import numpy as np

from .config import Camera
from .errors import ParseError, ValidationError
from .scene import DEFAULT_SIGMA_EPS, Scene

PLY_DT_REF = 0.01
S_MIN = 1e-7
N_SH, N_SG = 9, 7


# -- cameras -----------------------------------------------------------------
def _vec(n):
    def conv(v):
        a = np.asarray(v, dtype=float)
        if a.shape != (n,):
            raise ValueError(f"expected {n} numbers, got shape {a.shape}")
        return a
    return conv


# (JSON key, Camera attribute, parse, dump, default or None when required)
_CAMERA_SCHEMA = (
    ("center", "center", _vec(3), lambda v: [float(x) for x in v], None),
    ("quat", "quat", _vec(4), lambda v: [float(x) for x in v], None),
    ("focal_px", "focal", float, float, None),
    ("width", "width", int, int, None),
    ("height", "height", int, int, None),
    ("t_near", "t_near", float, float, 1e-4),
    ("t_far", "t_far", float, float, 1e6),
)


def camera_to_json(cam: Camera) -> dict:
    return {key: dump(getattr(cam, attr)) for key, attr, _, dump, _ in _CAMERA_SCHEMA}


def camera_from_json(entry: dict) -> Camera:
    kw = {}
    for key, attr, parse, _, default in _CAMERA_SCHEMA:
        if key in entry:
            kw[attr] = parse(entry[key])
        elif default is None:
            raise KeyError(f"camera entry lacks {key!r}")
        else:
            kw[attr] = default
    return Camera(**kw)


def save_cameras(cameras, path):
    doc = {"cameras": [camera_to_json(c) for c in cameras]}
    Path(path).write_text(json.dumps(doc, indent=2) + "\n")


def load_cameras(path) -> list:
    """Cameras of a JSON file; ParseError if unreadable, ValidationError
    (with the entry index as `record`) for a malformed entry or an empty list."""
    try:
        doc = json.loads(Path(path).read_text())
    except (OSError, json.JSONDecodeError) as e:
        raise ParseError(f"cannot read camera file: {e}") from e
    entries = doc.get("cameras", []) if isinstance(doc, dict) else []
    if not entries:
        raise ValidationError("camera file lists no cameras")
    out = []
    for idx, entry in enumerate(entries):
        try:
            out.append(camera_from_json(entry))
        except (KeyError, ValueError, TypeError) as e:
            raise ValidationError(str(e), record=idx) from e
    return out


# -- PLY ---------------------------------------------------------------------
_PLY_TYPES = {"float": "<f4", "float32": "<f4", "double": "<f8", "float64": "<f8"}
PLY_REQUIRED = ["x", "y", "z", "rot_0", "rot_1", "rot_2", "rot_3", "scale_0", "scale_1",
                "scale_2", "opacity", "f_dc_0", "f_dc_1", "f_dc_2"]


def _ply_header(blob: bytes):
    """(format, [(element name, count, [(property name, type)])], payload offset)."""
    if not blob.startswith(b"ply"):
        raise ParseError("not a PLY file")
    end = blob.find(b"end_header")
    if end < 0:
        raise ParseError("unexpected end of PLY header")
    body = blob.find(b"\n", end)
    body = len(blob) if body < 0 else body + 1
    fmt, elements = None, []
    for raw in blob[:end].decode("ascii", "replace").splitlines()[1:]:
        tok = raw.split()
        if not tok or tok[0] in ("comment", "obj_info"):
            continue
        if tok[0] == "format" and len(tok) > 1:
            fmt = tok[1]
        elif tok[0] == "element" and len(tok) > 2:
            elements.append((tok[1], int(tok[2]), []))
        elif tok[0] == "property" and elements:
            elements[-1][2].append((tok[-1], tok[1]))
    return fmt, elements, body


def read_ply_vertices(path):
    """Vertex table of a PLY file: (names, float64 [n, k]); float/double
    properties, ascii or binary little-endian (the subset scene_io.py:330-380
    accepts).  Only the vertex element is decoded; it must be the first
    element of the file."""
    blob = Path(path).read_bytes()
    fmt, elements, body = _ply_header(blob)
    if fmt not in ("ascii", "binary_little_endian"):
        raise ParseError(f"unsupported PLY format {fmt!r}")
    if not elements or elements[0][0] != "vertex" or not elements[0][2]:
        raise ParseError("PLY has no vertex element")
    _, count, props = elements[0]
    for _, t in props:
        if t not in _PLY_TYPES:
            raise ParseError(f"unsupported property type {t!r}")
    names = [nm for nm, _ in props]
    if fmt == "binary_little_endian":
        rec = np.dtype([(nm, _PLY_TYPES[t]) for nm, t in props])
        if len(blob) - body < rec.itemsize * count:
            raise ParseError("truncated PLY payload")
        table = np.frombuffer(blob, dtype=rec, count=count, offset=body)
        data = np.empty((count, len(names)), dtype=np.float64)
        for i, nm in enumerate(names):
            data[:, i] = table[nm]
        return names, data
    lines = blob[body:].decode("ascii", "replace").splitlines()
    rows = [ln for ln in lines if ln.strip()][:count]
    if len(rows) < count or any(len(ln.split()) != len(names) for ln in rows):
        raise ParseError("short PLY vertex row")
    data = np.loadtxt(io.StringIO("\n".join(rows)), dtype=np.float64, ndmin=2)
    return names, data.reshape(count, len(names))


def ply_records(path, sigma_eps: float = DEFAULT_SIGMA_EPS) -> np.ndarray:
    """[N,87] float32 records of a 3DGS PLY (vectorized scene_io.py:287-327)."""
    names, data = read_ply_vertices(Path(path))
    col = {n: data[:, i] for i, n in enumerate(names)}
    for r in PLY_REQUIRED:
        if r not in col:
            raise ParseError(f"PLY missing property {r!r}")
    n = data.shape[0]
    alpha = np.clip(1.0 / (1.0 + np.exp(-col["opacity"])), 1e-6, 1.0 - 1e-6)
    sigma = -np.log1p(-alpha) / PLY_DT_REF
    bad = np.nonzero(sigma <= sigma_eps)[0]
    if bad.size:
        i = int(bad[0])
        raise ValidationError(f"opacity maps to amplitude {sigma[i]:.3g} <= sigma_eps", record=i)
    rec = np.zeros((n, 87), dtype=np.float64)
    rec[:, 0] = col["x"]
    rec[:, 1] = col["y"]
    rec[:, 2] = col["z"]
    q = np.stack([col[f"rot_{k}"] for k in range(4)], axis=1)
    with np.errstate(invalid="ignore", divide="ignore"):
        rec[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)  # GaussianShape (geometry.py)
    rec[:, 7:10] = np.maximum(np.exp(np.stack([col[f"scale_{k}"] for k in range(3)], axis=1)),
                              S_MIN)
    rec[:, 10] = sigma
    rec[:, 11:14] = np.stack([col[f"f_dc_{k}"] for k in range(3)], axis=1)  # sh[0]
    rec[:, 40:59:3] = 1.0  # AppearanceCoeffs.constant: unit lobe axes (0, 0, 1)
    return rec.astype("<f4")


def load_ply_scene(path, sigma_eps: float = DEFAULT_SIGMA_EPS, device=None) -> Scene:
    """Ingest a 3DGS-style PLY point cloud (scene_io.py:287-327) onto the
    device: x/y/z, rot_0..3 (scalar first), scale_0..2 (log scales), opacity
    (pre-sigmoid), f_dc_0..2 (SH DC)."""
    return Scene.from_records(ply_records(path, sigma_eps), sigma_eps=sigma_eps, device=device)
