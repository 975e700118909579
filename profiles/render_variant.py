"""One forward of a workload with a given renderer variant, for ncu:
    ncu ... -k regex:"k_render_(camera|screened)" --launch-skip 1 -c 1 \
        python profiles/render_variant.py c3 screened-regs [logged]
("logged": the training forward, recording a march log)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_07782_b200 as G  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
variant = sys.argv[2] if len(sys.argv) > 2 else "plain"
rec, eps, cam_kw, cfg_kw, desc = bench.workload(cfgname)
scene = G.Scene.from_records(rec)
G.reorder_by_morton(scene)
cam = bench.make_camera(G, cam_kw)
cfg = G.RenderConfig(**cfg_kw)
log = None
if len(sys.argv) > 3 and sys.argv[3] == "logged":
    from paper_2509_07782_b200.renderer import MarchLog
    log = MarchLog(cam)
for _ in range(2):
    G.render(scene, cam, cfg, variant=variant, log=log)
torch.cuda.synchronize()
print("ok")
