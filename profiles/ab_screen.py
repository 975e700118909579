"""A/B of the plain camera forward with and without the silhouette screen
(render(screen=...)): median device ms over 7 L2-flushed renders after 2
warm-ups, per workload, and the max |rgb| / |T| difference between the two.

    python profiles/ab_screen.py [c3 c2 ...]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_07782_b200 as G  # noqa: E402


def timed(fn, reps=7, warm=2):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(reps + warm):
        flush.zero_()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        out = fn()
        e1.record(s)
        torch.cuda.synchronize()
        if i >= warm:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), out


for name in sys.argv[1:] or ["c3", "c2"]:
    rec, eps, cam_kw, cfg_kw, desc = bench.workload(name)
    scene = G.Scene.from_records(rec)
    G.reorder_by_morton(scene)
    cam = bench.make_camera(G, cam_kw)
    cfg = G.RenderConfig(**cfg_kw)
    res = {"config": name}
    outs = {}
    for label, kw in (("plain", dict(screen=False)), ("screen", dict(screen=True)),
                      ("screen_cone", dict(screen=True, traversal=1))):
        ms, (rgb, depth, trans, _) = timed(lambda: G.render(scene, cam, cfg, **kw))
        res[label + "_ms"] = ms
        outs[label] = (rgb.clone(), trans.clone())
    for label in ("screen", "screen_cone"):
        res[label + "_maxdiff_rgb"] = float((outs[label][0] - outs["plain"][0]).abs().max())
        res[label + "_maxdiff_T"] = float((outs[label][1] - outs["plain"][1]).abs().max())
    print(json.dumps(res), flush=True)
    del scene
    torch.cuda.empty_cache()
