"""A/B of the training step's logged forward with and without the
silhouette screen (render(..., log=, screen=)), and the logged backward that
consumes each log, on C2 (and C4 with `c4`): median device ms over 5 runs.

    python profiles/ab_train.py [c2|c4]
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

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
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


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


res = {"config": name}
for screen in (False, True):
    key = "screen" if screen else "plain"
    res[key + "_fwd_logged_ms"] = timed(lambda: G.render(scene, cam, cfg, rgb=tr.rgb,
                                                           depth=tr.depth, trans=tr.trans,
                                                           log=tr.log, screen=screen))
    used, ovf = tr.log.usage()
    res[key + "_log_bytes"] = used
    tr.loss(tr.rgb, target, tr.loss_cfg.mix, grad=tr.dI, want_value=False)

    def bwd():
        tr.grad.zero_()
        G.render_backward(scene, cam, cfg, tr.rgb, tr.depth, tr.trans, tr.dI, grad=tr.grad,
                          log=tr.log)

    res[key + "_bwd_logged_ms"] = timed(bwd)
    g = tr.grad.clone()
    res[key + "_grad_norm"] = float(g.norm())
    for p2, p2name in ((1, "pairs"), (2, "entries")):  # forced pass-2 strategy
        res[key + "_bwd_logged_" + p2name + "_ms"] = timed(
            lambda: G.render_backward(scene, cam, cfg, tr.rgb, tr.depth, tr.trans, tr.dI,
                                      grad=tr.grad, log=tr.log, pass2=p2))
res["fwd_unlogged_ms"] = timed(lambda: G.render(scene, cam, cfg))
res["step_ms"] = timed(lambda: tr.step(target))
print(json.dumps(res), flush=True)
