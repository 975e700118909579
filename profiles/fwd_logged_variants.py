"""Steady-state device ms of the logged training forward per kernel variant
(the autotuner's pick is timed once, on the first frames):

    python profiles/fwd_logged_variants.py c4 c2
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_07782_b200 as G  # noqa: E402
from paper_2509_07782_b200.train import Trainer  # noqa: E402

for name in sys.argv[1:] or ["c4"]:
    rec, eps, cam_kw, cfg_kw, desc = bench.workload(name)
    cam = bench.make_camera(G, cam_kw)
    cfg = G.RenderConfig(**cfg_kw)
    scene = G.Scene.from_records(rec)
    G.reorder_by_morton(scene)
    target = G.render(scene, cam, cfg)[0].clone()
    tr = Trainer(scene, cam, cfg)
    for _ in range(3):
        tr.step(target)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    out = {"config": name}
    for variant in ("screened", "screened-regs", "plain"):
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            G.render(scene, cam, cfg, rgb=tr.rgb, depth=tr.depth, trans=tr.trans, log=tr.log,
                     variant=variant)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[variant] = round(float(np.median(ts[2:])), 3)
    print(json.dumps(out), flush=True)
