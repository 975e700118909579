"""Experiment: how much does BVH quality cost the C3 forward?  Builds a
binned-SAH binary BVH (profiles/experiments/sah_bvh.c, CPU, single-primitive
leaves) over the same fp32 leaf boxes as the device LBVH, loads it into the
scene's BVH arena, re-derives the 4-wide nodes (gsx_bvh_collapse) and times
the same render.  Not product code.

    gcc -O2 -shared -fPIC -o /tmp/libsah.so profiles/experiments/sah_bvh.c -lm
    python profiles/experiments/sah_vs_lbvh.py /tmp/libsah.so
"""
import ctypes
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_07782_b200 as G  # noqa: E402
from paper_2509_07782_b200 import _lib  # noqa: E402
from paper_2509_07782_b200._lib import check, ptr  # noqa: E402


def timed_render(scene, cam, cfg, reps=5):
    G.render(scene, cam, cfg)
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        G.render(scene, cam, cfg)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    _, _, _, st = G.render(scene, cam, cfg, stats=True)
    c = st.cpu().numpy()
    return float(np.median(ts)), float(c[5] / max(c[0], 1))


def main(libpath, cfgname="c3"):
    rec, eps, cam_kw, cfg_kw, desc = bench.workload(cfgname)
    scene = G.Scene.from_records(rec)
    G.reorder_by_morton(scene)
    cam = bench.make_camera(G, cam_kw)
    cfg = G.RenderConfig(**cfg_kw)
    out = {"config": cfgname}
    out["lbvh_ms"], out["lbvh_node_visits_per_ray"] = timed_render(scene, cam, cfg)
    n = scene.n
    L = _lib.lib()
    m = n - 1
    boxes = torch.empty((m, 12), dtype=torch.float32, device="cuda")
    children = torch.empty((m, 2), dtype=torch.int32, device="cuda")
    check(L.gsx_bvh_export(ptr(scene.bvh_arena), n, ptr(boxes), ptr(children), None, None))
    torch.cuda.synchronize()
    b = boxes.cpu().numpy()
    c = children.cpu().numpy()
    lo = np.zeros((n, 3), np.float32)
    hi = np.zeros((n, 3), np.float32)
    for side in (0, 1):
        leaf = c[:, side] < 0
        prim = ~c[leaf, side]
        lo[prim] = b[leaf, 6 * side:6 * side + 3]
        hi[prim] = b[leaf, 6 * side + 3:6 * side + 6]
    sah = ctypes.CDLL(libpath)
    nodes = np.zeros((m, 16), np.float32)
    parents = np.zeros(2 * n + 1, np.int32)
    t0 = time.time()
    sah.sah_build(ctypes.c_int64(n), lo.ctypes.data_as(ctypes.c_void_p),
                  hi.ctypes.data_as(ctypes.c_void_p), nodes.ctypes.data_as(ctypes.c_void_p),
                  parents.ctypes.data_as(ctypes.c_void_p))
    out["sah_build_s_cpu"] = time.time() - t0
    arena = scene.bvh_arena
    nb = nodes.nbytes
    arena[:nb].copy_(torch.from_numpy(nodes.view(np.uint8).ravel()))
    off = (nb + 255) & ~255
    pb = parents.view(np.uint8).ravel()
    arena[off:off + pb.size].copy_(torch.from_numpy(pb))
    check(L.gsx_bvh_collapse(ptr(arena), n, ptr(scene._bvh_ws), None), "collapse")
    torch.cuda.synchronize()
    out["sah_ms"], out["sah_node_visits_per_ray"] = timed_render(scene, cam, cfg)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "c3")
