"""C-ABI checks on CPU (no GPU needed): libgsx.so loads, exports every symbol
include/gsx.h declares, and the ctypes table matches the header; host-side
config mirrors validate like the reference."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def header_functions():
    src = (ROOT / "include" / "gsx.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gsx_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2509_07782_b200 import _lib

    L = _lib.load_library()
    funcs = header_functions()
    assert len(funcs) >= 25
    for f in funcs:
        assert hasattr(L, f), f
    assert sorted(_lib.EXPORTED) == funcs
    assert L.gsx_abi_version() == 3
    assert L.gsx_status_string(0) == b"ok"
    assert L.gsx_scene_arena_bytes(1000) > 1000 * 87 * 4
    assert L.gsx_sort_workspace_bytes(1 << 20) > 0


def test_size_queries_and_argument_errors_without_gpu():
    from paper_2509_07782_b200 import _lib

    L = _lib.load_library()
    # argument validation happens before any CUDA call
    assert L.gsx_prepare(None, 0, 0.01, None, None, None, None) == _lib.GSX_ERR_EMPTY
    assert L.gsx_prepare(ctypes.c_void_p(8), 4, -1.0, ctypes.c_void_p(8), None, None,
                         None) == _lib.GSX_ERR_ARG
    cfg = _lib.RenderCfg()
    cfg.dt, cfg.n_s, cfg.t_eps, cfg.mode = 0.0025, 16, 0.0, 0
    cam = _lib.CameraC()
    cam.width = cam.height = 4
    cam.focal = 1.0
    rc = L.gsx_render_forward(None, None, 10, ctypes.byref(cam), ctypes.byref(cfg), 0, 1, None,
                              None, None, None, None, 0, None, None)
    assert rc == _lib.GSX_ERR_ARG  # t_eps must be in (0, 1)
    cfg.t_eps = 1e-4
    for field, bad in (("traversal", 3), ("sums", 2), ("pass2", 3), ("pass2", -1)):
        setattr(cfg, field, bad)
        rc = L.gsx_render_forward(None, None, 10, ctypes.byref(cam), ctypes.byref(cfg), 0, 1,
                                  None, None, None, None, None, 0, None, None)
        assert rc == _lib.GSX_ERR_ARG, field  # extension fields are range-checked
        setattr(cfg, field, 0)
    assert L.gsx_image_loss(None, None, 8, 8, 3, 0.2, None, None, None, None) == _lib.GSX_ERR_ARG


def test_config_mirrors():
    from paper_2509_07782_b200 import Camera, RenderConfig, segment_step

    with pytest.raises(ValueError):
        RenderConfig(mode="fancy")
    with pytest.raises(ValueError):
        RenderConfig(t_eps=0.0)
    with pytest.raises(ValueError):
        RenderConfig(dt_min=0.1, dt_max=0.01)
    with pytest.raises(ValueError):
        Camera(center=[0, 0, 0], quat=[1, 0, 0, 0], focal=0.0, width=4, height=4)
    cfg = RenderConfig(mode="adaptive", beta=1024, dt_min=0.005, dt_max=0.02, n_s=16)
    assert segment_step(cfg, 10.24, 0.125) == pytest.approx(0.32, abs=1e-12)
    c = cfg.to_c()
    assert c.mode == 1 and c.n_s == 16 and c.ess == 1


def test_product_package_fails_loudly_without_gpu():
    import torch

    import paper_2509_07782_b200 as G
    from paper_2509_07782_b200 import _lib

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.GsxUnavailable):
        G.Scene.from_records([[0.0] * 87])


def test_camera_rays_vectorised_matches_ray():
    import numpy as np

    import paper_2509_07782_b200 as G

    cam = G.orbit_cameras(2, radius=3.5, focal=40.0, width=9, height=7)[1]
    r = cam.rays()
    assert r.shape == (63, 8)
    for py, px in ((0, 0), (3, 5), (6, 8)):
        one = cam.ray(px, py)
        np.testing.assert_array_equal(r[py * 9 + px, 0:3], one.origin)
        np.testing.assert_allclose(r[py * 9 + px, 3:6], one.direction, rtol=0, atol=1e-15)


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors in _lib.py have the size and field offsets of the
    C structs in include/gsx.h (compiled here with gcc)."""
    import shutil
    import subprocess

    from paper_2509_07782_b200 import _lib

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    root = Path(__file__).resolve().parent.parent
    checks = {
        "gsx_render_cfg": (_lib.RenderCfg, ["dt", "n_s", "t_eps", "mode", "background",
                                             "buffer_capacity", "traversal", "sums", "pass2"]),
        "gsx_camera": (_lib.CameraC, [f for f, _ in _lib.CameraC._fields_]),
        "gsx_stats": (_lib.Stats, ["rays", "composited"]),
    }
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "gsx.h"', "int main(void) {"]
    for st, (_, fields) in checks.items():
        lines.append(f'  printf("{st} size %zu\\n", sizeof({st}));')
        for f in fields:
            lines.append(f'  printf("{st} {f} %zu\\n", offsetof({st}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(root / "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    got = {}
    for line in out.splitlines():
        st, key, val = line.split()
        got[(st, key)] = int(val)
    for st, (cls, fields) in checks.items():
        assert got[(st, "size")] == ctypes.sizeof(cls), st
        for f in fields:
            assert got[(st, f)] == getattr(cls, f).offset, (st, f)
