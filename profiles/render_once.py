"""One C3 (or C1/C2) forward render for ncu captures:
    ncu --set full --import-source on -k regex:k_render_camera --launch-skip 1 -c 1 \
        -o OUT python profiles/render_once.py c3
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_07782_b200 as G  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
rec, eps, cam_kw, cfg_kw, desc = bench.workload(cfgname)
scene = G.Scene.from_records(rec)
G.reorder_by_morton(scene)
cam = bench.make_camera(G, cam_kw)
cfg = G.RenderConfig(**cfg_kw)
for _ in range(2):
    G.render(scene, cam, cfg)
torch.cuda.synchronize()
print("ok")
