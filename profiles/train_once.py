"""Two C2 (or C4) training steps for ncu captures of the logged forward and
the logged backward:
    ncu --set full --import-source on -k regex:"k_render_camera|k_render_backward_logged" \
        --launch-skip 3 -c 2 -o OUT python profiles/train_once.py c2
(launches: target render, warm-up step's forward + backward, then the step)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_07782_b200 as G  # noqa: E402
from paper_2509_07782_b200.train import Trainer  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
rec, eps, cam_kw, cfg_kw, desc = bench.workload(cfgname)
cam = bench.make_camera(G, cam_kw)
cfg = G.RenderConfig(**cfg_kw)
tscene = G.Scene.from_records(rec)
G.reorder_by_morton(tscene)
target = G.render(tscene, cam, cfg)[0].clone()
jit = tscene.records().copy()
base = 0.08 * (32.0 / rec.shape[0]) ** (1.0 / 3.0)
jit[:, 0:3] += np.random.default_rng(1).normal(0, 0.1 * base, size=(jit.shape[0], 3))
scene = G.Scene.from_records(jit.astype(np.float32))
del tscene
tr = Trainer(scene, cam, cfg)
for _ in range(2):
    tr.step(target)
torch.cuda.synchronize()
print("ok")
