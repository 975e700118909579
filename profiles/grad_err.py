"""Error structure of the C2 (or C4) backward (sparse pixel mask) against
the float64 oracle backward: per parameter group, the relative error of the
entries by magnitude bin (|g| / max|g| of the group), for the replay and
the logged backward (both pass-2 strategies).

    python profiles/grad_err.py [c2|c4] > gpurun_out/grad_err.json
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from test_gpu_bench_parity import _pixels, _setup  # noqa: E402

CFG = sys.argv[1] if len(sys.argv) > 1 else "c2"
G, rec, eps, scene, cam, cfg, cfg_kw = _setup(CFG)
H, W = cam.height, cam.width
rays, py, px = _pixels(cam, *((40, 17, 23) if CFG == "c2" else (64, 21, 29)))
rng = np.random.default_rng(3)
gC = np.zeros((H, W, 3)); gT = np.zeros((H, W)); gD = np.zeros((H, W))
gC[py, px] = rng.normal(size=(len(py), 3))
gT[py, px] = rng.normal(size=len(py))
gD[py, px] = 0.1 * rng.normal(size=len(py))
t = lambda a: torch.as_tensor(a, dtype=torch.float32, device="cuda")  # noqa: E731
osc = O.OracleScene(rec, eps)
_, _, _, g_ref = osc.backward_rays(rays, O.OCfg.make(**cfg_kw), gC[py, px], gD[py, px],
                                   gT[py, px], clip=True)
uids = scene.uids
res = {}
for log, pass2 in ((None, 0), ("full", 1), ("full", 2)):
    lg = None
    if log:
        lg = G.MarchLog(cam)
        for _ in range(2):
            G.render(scene, cam, cfg, log=lg)
            if not lg.ensure():
                break
    rgb, depth, trans, _ = G.render(scene, cam, cfg, log=lg)
    g = G.render_backward(scene, cam, cfg, rgb, depth, trans, t(gC), t(gD), t(gT), log=lg,
                          pass2=pass2)
    g_gpu = np.empty_like(g_ref)
    g_gpu[uids] = g.cpu().numpy()
    out = {}
    for name, (a, b) in {"mean": (0, 3), "quat": (3, 7), "scale": (7, 10), "sigma": (10, 11),
                         "sh": (11, 38), "axis": (38, 59), "sharp": (59, 66),
                         "amp": (66, 87)}.items():
        A, B = g_gpu[:, a:b].ravel(), g_ref[:, a:b].ravel()
        gmax = np.abs(B).max()
        rel = np.abs(A - B) / np.maximum(np.abs(B), 1e-300)
        absn = np.abs(A - B) / gmax
        bins = {}
        for lo, hi in ((1e-1, 1.1), (1e-2, 1e-1), (1e-3, 1e-2), (1e-4, 1e-3), (0, 1e-4)):
            m = (np.abs(B) / gmax >= lo) & (np.abs(B) / gmax < hi) & (B != 0)
            if m.any():
                bins[f"{lo:g}-{hi:g}"] = {"n": int(m.sum()), "rel_max": float(rel[m].max()),
                                          "rel_p99": float(np.quantile(rel[m], 0.99)),
                                          "abs_over_gmax_max": float(absn[m].max())}
        out[name] = {"gmax": float(gmax), "abs_over_gmax_max": float(absn.max()), "bins": bins}
    res[f"{log}/pass2={pass2}"] = out
print(json.dumps(res, indent=1))
