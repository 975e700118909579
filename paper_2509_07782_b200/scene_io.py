"""Scene / camera file ingestion (scene_io.py of the reference).

* `.gsx` records: `scene.save_scene` / `scene.load_scene` (bit-exact).
* Cameras JSON: `save_cameras` / `load_cameras` (scene_io.py:114-155), same
  file layout and errors.
* 3DGS PLY: `load_ply_scene` (scene_io.py:287-327) parses the vertex table
  with numpy (ascii or binary little-endian, scene_io.py:330-380), converts
  all rows at once to the 87-float record layout exactly as the reference's
  GaussianShape / AppearanceCoeffs ingestion does (quaternion normalized in
  float64, scales exp'd and clamped at S_MIN, sigma~ = -ln(1 - alpha)/dt_ref
  with alpha = clip(sigmoid(opacity), 1e-6, 1 - 1e-6), SH DC from f_dc, lobes
  of `AppearanceCoeffs.constant`), and hands the [N,87] float32 block to the
  device in one copy (`Scene.from_records`).
* `export_density_ply` (scene_io.py:383-398).
"""

from __future__ import annotations

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
def save_cameras(cameras, path):
    out = {"cameras": [{"center": list(map(float, c.center)), "quat": list(map(float, c.quat)),
                        "focal_px": c.focal, "width": c.width, "height": c.height,
                        "t_near": c.t_near, "t_far": c.t_far} for c in cameras]}
    Path(path).write_text(json.dumps(out, indent=2) + "\n")


def load_cameras(path) -> list:
    try:
        data = json.loads(Path(path).read_text())
    except (OSError, json.JSONDecodeError) as e:
        raise ParseError(f"cannot read camera file: {e}") from e
    cams = []
    for i, c in enumerate(data.get("cameras", [])):
        try:
            cams.append(Camera(center=np.asarray(c["center"], dtype=float),
                               quat=np.asarray(c["quat"], dtype=float),
                               focal=float(c["focal_px"]), width=int(c["width"]),
                               height=int(c["height"]), t_near=float(c.get("t_near", 1e-4)),
                               t_far=float(c.get("t_far", 1e6))))
        except (KeyError, ValueError) as e:
            raise ValidationError(str(e), record=i) from e
    if not cams:
        raise ValidationError("camera file lists no cameras")
    return cams


# -- PLY ---------------------------------------------------------------------
_PLY_SIZES = {b"float": "<f4", b"float32": "<f4", b"double": "<f8", b"float64": "<f8"}
PLY_REQUIRED = ["x", "y", "z", "rot_0", "rot_1", "rot_2", "rot_3", "scale_0", "scale_1",
                "scale_2", "opacity", "f_dc_0", "f_dc_1", "f_dc_2"]


def read_ply_vertices(path):
    """Vertex table of a PLY file: (names, float64 [n, k]); float/double
    properties, ascii or binary little-endian (scene_io.py:330-380)."""
    with open(path, "rb") as f:
        if f.readline().strip() != b"ply":
            raise ParseError("not a PLY file")
        fmt, n_vertex, names, types = None, None, [], []
        while True:
            line = f.readline()
            if not line:
                raise ParseError("unexpected end of PLY header")
            parts = line.split()
            if not parts:
                continue
            if parts[0] == b"format":
                fmt = parts[1]
            elif parts[0] == b"element":
                if parts[1] == b"vertex":
                    n_vertex = int(parts[2])
                elif n_vertex is not None:
                    break  # only the vertex element is read
            elif parts[0] == b"property" and n_vertex is not None:
                if parts[1] not in _PLY_SIZES:
                    raise ParseError(f"unsupported property type {parts[1]!r}")
                types.append(parts[1])
                names.append(parts[2].decode())
            elif parts[0] == b"end_header":
                break
        if fmt not in (b"ascii", b"binary_little_endian"):
            raise ParseError(f"unsupported PLY format {fmt!r}")
        if n_vertex is None or not names:
            raise ParseError("PLY has no vertex element")
        if fmt == b"ascii":
            rows = []
            for _ in range(n_vertex):
                vals = f.readline().split()
                if len(vals) != len(names):
                    raise ParseError("short PLY vertex row")
                rows.append([float(v) for v in vals])
            data = np.array(rows, dtype=np.float64).reshape(n_vertex, len(names))
        else:
            dtype = np.dtype([(nm, _PLY_SIZES[t]) for nm, t in zip(names, types)])
            raw = np.frombuffer(f.read(dtype.itemsize * n_vertex), dtype=dtype)
            if raw.shape[0] != n_vertex:
                raise ParseError("truncated PLY payload")
            data = np.stack([raw[nm].astype(np.float64) for nm in names], axis=1)
    return names, data


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


def export_density_ply(path, means, counts):
    """ASCII PLY point cloud with a per-point neighbor-count scalar."""
    means = np.asarray(means, dtype=float).reshape(-1, 3)
    counts = np.asarray(counts).reshape(-1)
    lines = ["ply", "format ascii 1.0", f"element vertex {len(means)}", "property float x",
             "property float y", "property float z", "property float density", "end_header"]
    for m, c in zip(means, counts):
        lines.append(f"{m[0]} {m[1]} {m[2]} {float(c)}")
    Path(path).write_text("\n".join(lines) + "\n")
