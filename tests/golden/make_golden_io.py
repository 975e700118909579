"""Golden vectors for scene / camera ingestion, from the REFERENCE.

Run in the build container only (imports /root/reference/pkg/src):

    python tests/golden/make_golden_io.py

Writes io.npz: a random 3DGS PLY (binary little-endian, 300 vertices, with an
extra unused property) and an ascii PLY, their bytes, the reference's
load_ply_scene records (scene_io.py:287-327 -> _record, float32), and a
camera JSON written by the reference's save_cameras.
"""

from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from gsray.scene_io import _record, load_ply_scene, orbit_cameras, save_cameras  # noqa: E402

NAMES = ["x", "y", "z", "nx", "rot_0", "rot_1", "rot_2", "rot_3", "scale_0", "scale_1",
         "scale_2", "opacity", "f_dc_0", "f_dc_1", "f_dc_2"]


def header(fmt, n):
    props = "".join(f"property float {nm}\n" for nm in NAMES)
    return f"ply\nformat {fmt} 1.0\nelement vertex {n}\n{props}end_header\n"


def main():
    rng = np.random.default_rng(11)
    n = 300
    cols = {
        "x": rng.uniform(-2, 2, n), "y": rng.uniform(-2, 2, n), "z": rng.uniform(-2, 2, n),
        "nx": rng.normal(size=n),
        "rot_0": rng.normal(size=n), "rot_1": rng.normal(size=n), "rot_2": rng.normal(size=n),
        "rot_3": rng.normal(size=n),
        "scale_0": rng.uniform(-7, -2, n), "scale_1": rng.uniform(-7, -2, n),
        "scale_2": rng.uniform(-20, -2, n),  # some below S_MIN after exp
        "opacity": rng.uniform(-3, 6, n),
        "f_dc_0": rng.normal(size=n), "f_dc_1": rng.normal(size=n), "f_dc_2": rng.normal(size=n),
    }
    table = np.stack([cols[k] for k in NAMES], axis=1).astype("<f4")
    binary = header("binary_little_endian", n).encode() + table.tobytes()
    ascii_rows = table[:20].astype(np.float64)
    ascii_ply = header("ascii", 20) + "".join(
        " ".join(repr(float(v)) for v in r) + "\n" for r in ascii_rows)
    out = {"ply_binary": np.frombuffer(binary, dtype=np.uint8),
           "ply_ascii": np.frombuffer(ascii_ply.encode(), dtype=np.uint8)}
    with tempfile.TemporaryDirectory() as td:
        for key, data in (("binary", binary), ("ascii", ascii_ply.encode())):
            p = Path(td) / f"{key}.ply"
            p.write_bytes(data)
            sc = load_ply_scene(p)
            out[f"records_{key}"] = np.stack([_record(s, c) for s, c in
                                              zip(sc.shapes, sc.coeffs)])
        cams = orbit_cameras(3, radius=4.0, focal=500.0, width=640, height=480)
        p = Path(td) / "cams.json"
        save_cameras(cams, p)
        out["cameras_json"] = np.frombuffer(p.read_bytes(), dtype=np.uint8)
        out["cameras_center"] = np.stack([c.center for c in cams])
        out["cameras_quat"] = np.stack([c.quat for c in cams])
    np.savez_compressed(OUT / "io.npz", **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
