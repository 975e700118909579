"""renderer.autotune on the benchmark workloads: device ms of every forward
variant (screened / screened-regs / plain) per workload, one JSON line each.
Run with GSX_LIB=... to compare library builds on one box.

    python profiles/tune_report.py c3 c4 c2
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_07782_b200 as G  # noqa: E402

for name in sys.argv[1:] or ["c3"]:
    rec, eps, cam_kw, cfg_kw, desc = bench.workload(name)
    scene = G.Scene.from_records(rec)
    G.reorder_by_morton(scene)
    cam = bench.make_camera(G, cam_kw)
    cfg = G.RenderConfig(**cfg_kw)
    res = G.autotune(scene, cam, cfg, reps=5)
    res = {"config": name, "lib": Path(os.environ.get("GSX_LIB", "libgsx.so")).name,
           **{k: (round(v, 3) if isinstance(v, float) else v) for k, v in res.items()}}
    print(json.dumps(res), flush=True)
    del scene
    torch.cuda.empty_cache()
