"""Scene / camera ingestion (paper_2509_07782_b200/scene_io.py) against the
reference's scene_io.py: tests/golden/io.npz (tests/golden/make_golden_io.py)
holds PLY files and the records the reference's load_ply_scene produced, and
a camera file written by the reference's save_cameras.  Host-side parsing
only (CPU); device ingestion is covered in test_gpu_edge.py."""

import json
import math

import numpy as np
import pytest

from conftest import golden
from paper_2509_07782_b200 import scene_io as S
from paper_2509_07782_b200.errors import ParseError, ValidationError


@pytest.mark.parametrize("kind", ["binary", "ascii"])
def test_ply_records_bit_exact_vs_reference(kind, tmp_path):
    g = golden("io")
    p = tmp_path / f"{kind}.ply"
    p.write_bytes(g[f"ply_{kind}"].tobytes())
    rec = S.ply_records(p)
    ref = g[f"records_{kind}"]
    assert rec.dtype == np.float32 and rec.shape == ref.shape
    assert np.array_equal(rec.view(np.uint32), ref.view(np.uint32))


PLY_HEADER = """ply
format ascii 1.0
element vertex {n}
property float x
property float y
property float z
property float rot_0
property float rot_1
property float rot_2
property float rot_3
property float scale_0
property float scale_1
property float scale_2
property float opacity
property float f_dc_0
property float f_dc_1
property float f_dc_2
end_header
"""


def _write(path, rows):
    path.write_text(PLY_HEADER.format(n=len(rows)) +
                    "\n".join(" ".join(str(v) for v in r) for r in rows) + "\n")


def test_ply_ingest_values(tmp_path):
    """test_scene_io.py TestPly.test_ingest."""
    p = tmp_path / "cloud.ply"
    ls = math.log(0.1)
    _write(p, [[0.1, 0.2, 0.3, 1, 0, 0, 0, ls, ls, ls, 2.0, 0.5, 0.4, 0.3],
               [1.0, 1.0, 1.0, 0, 0, 0, 1, ls, ls, ls, 0.0, 0.1, 0.1, 0.1]])
    rec = S.ply_records(p)
    assert rec.shape == (2, 87)
    assert np.allclose(rec[0, 0:3], [0.1, 0.2, 0.3])
    assert np.allclose(rec[0, 7:10], 0.1)
    alpha = 1.0 / (1.0 + math.exp(-2.0))
    assert rec[0, 10] == pytest.approx(-math.log1p(-alpha) / 0.01, rel=1e-6)


def test_ply_binary_matches_ascii(tmp_path):
    ls = math.log(0.05)
    row = [0.1, -0.2, 0.3, 0.9, 0.1, 0.0, 0.0, ls, ls, ls, 1.5, 0.5, 0.4, 0.3]
    a = tmp_path / "a.ply"
    _write(a, [row])
    b = tmp_path / "b.ply"
    header = PLY_HEADER.format(n=1).replace("ascii 1.0", "binary_little_endian 1.0")
    b.write_bytes(header.encode() + np.array(row, dtype="<f4").tobytes())
    ra, rb = S.ply_records(a), S.ply_records(b)
    assert np.allclose(ra, rb, rtol=1e-6, atol=1e-7)


def test_ply_errors(tmp_path):
    p = tmp_path / "bad.ply"
    p.write_text("ply\nformat ascii 1.0\nelement vertex 1\nproperty float x\nproperty float y\n"
                 "property float z\nend_header\n0 0 0\n")
    with pytest.raises(ParseError):
        S.ply_records(p)
    p.write_text("hello\n")
    with pytest.raises(ParseError):
        S.ply_records(p)
    p.write_text("ply\nformat binary_big_endian 1.0\nelement vertex 1\nproperty float x\n"
                 "end_header\n")
    with pytest.raises(ParseError):
        S.ply_records(p)
    # opacity -> amplitude <= sigma_eps is a ValidationError naming the record
    ls = math.log(0.1)
    _write(p, [[0, 0, 0, 1, 0, 0, 0, ls, ls, ls, 2.0, 0, 0, 0],
               [0, 0, 0, 1, 0, 0, 0, ls, ls, ls, -20.0, 0, 0, 0]])
    with pytest.raises(ValidationError) as e:
        S.ply_records(p)
    assert e.value.record == 1


def test_ply_reader_header_forms(tmp_path):
    # comments, a trailing face element and a truncated binary payload
    p = tmp_path / "v.ply"
    p.write_text("ply\nformat ascii 1.0\ncomment made by hand\nelement vertex 3\n"
                 "property float x\nproperty float y\nproperty float z\n"
                 "property float density\nelement face 0\n"
                 "property list uchar int vertex_indices\nend_header\n"
                 "0 0 0 1\n0 0 0 2\n0 0 0 3\n")
    names, data = S.read_ply_vertices(p)
    assert names == ["x", "y", "z", "density"] and data[:, 3].tolist() == [1.0, 2.0, 3.0]
    b = tmp_path / "t.ply"
    b.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 2\n"
                  b"property float x\nend_header\n" + np.zeros(1, "<f4").tobytes())
    with pytest.raises(ParseError):
        S.read_ply_vertices(b)


def test_cameras_reference_file_and_roundtrip(tmp_path):
    g = golden("io")
    p = tmp_path / "cams.json"
    p.write_bytes(g["cameras_json"].tobytes())
    cams = S.load_cameras(p)
    assert len(cams) == 3
    np.testing.assert_array_equal(np.stack([c.center for c in cams]), g["cameras_center"])
    np.testing.assert_array_equal(np.stack([c.quat for c in cams]), g["cameras_quat"])
    q = tmp_path / "again.json"
    S.save_cameras(cams, q)
    assert json.loads(q.read_text()) == json.loads(p.read_text())


def test_camera_errors(tmp_path):
    p = tmp_path / "c.json"
    p.write_text("{not json")
    with pytest.raises(ParseError):
        S.load_cameras(p)
    p.write_text(json.dumps({"cameras": []}))
    with pytest.raises(ValidationError):
        S.load_cameras(p)
    p.write_text(json.dumps({"cameras": [{"center": [0, 0, 0]}]}))
    with pytest.raises(ValidationError) as e:
        S.load_cameras(p)
    assert e.value.record == 0
