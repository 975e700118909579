"""Time the logged backward (and the logged forward that feeds it) of one
training workload for several libgsx builds, one process per variant:

    python profiles/time_bwd_variants.py c2 lib_a.so lib_b.so ...

Prints one line per variant: median ms of the logged backward over 7 steps
after warm-up (L2 flushed before each) and the max relative |grad - first
variant's grad| (atomics reorder the sums, so ~1e-6 is noise).
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

if len(sys.argv) > 2 and sys.argv[1] == "--one":
    cfgname, out = sys.argv[2], sys.argv[3]
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import torch
    import bench
    import paper_2509_07782_b200 as G
    from paper_2509_07782_b200.renderer import MarchLog, render, render_backward
    from paper_2509_07782_b200.loss import ImageLoss

    rec, eps, cam_kw, cfg_kw, desc = bench.workload(cfgname)
    scene = G.Scene.from_records(rec)
    G.reorder_by_morton(scene)
    cam = bench.make_camera(G, cam_kw)
    cfg = G.RenderConfig(**cfg_kw)
    target = G.render(scene, cam, cfg)[0].clone()
    jit = scene.records().copy()
    base = 0.08 * (32.0 / rec.shape[0]) ** (1.0 / 3.0)
    jit[:, 0:3] += np.random.default_rng(1).normal(0, 0.1 * base, size=(jit.shape[0], 3))
    scene = G.Scene.from_records(jit.astype(np.float32))
    H, W = cam.height, cam.width
    dev = scene.device
    rgb = torch.zeros((H, W, 3), device=dev)
    depth = torch.zeros((H, W), device=dev)
    trans = torch.zeros((H, W), device=dev)
    dI = torch.empty((H, W, 3), device=dev)
    grad = torch.zeros_like(scene.params)
    loss = ImageLoss(H, W, 3, dev)
    log = MarchLog(cam, device=dev)
    render(scene, cam, cfg, rgb=rgb, depth=depth, trans=trans, log=log)
    log.ensure()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tf, tb = [], []
    s = torch.cuda.current_stream()
    for i in range(9):
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(s)
        render(scene, cam, cfg, rgb=rgb, depth=depth, trans=trans, log=log)
        e[1].record(s)
        loss(rgb, target, 0.2, grad=dI, want_value=False)
        grad.zero_()
        flush.zero_()
        e[2].record(s)
        render_backward(scene, cam, cfg, rgb, depth, trans, dI, grad=grad, log=log)
        e[3].record(s)
        torch.cuda.synchronize()
        if i >= 2:
            tf.append(e[0].elapsed_time(e[1]))
            tb.append(e[2].elapsed_time(e[3]))
    np.save(out, grad.cpu().numpy())
    print(json.dumps({"bwd_ms": float(np.median(tb)), "bwd_min": float(min(tb)),
                      "fwd_logged_ms": float(np.median(tf))}))
    sys.exit(0)

cfgname, libs = sys.argv[1], sys.argv[2:]
import numpy as np  # noqa: E402
first = None
for lib in libs:
    env = dict(os.environ, GSX_LIB=str(Path(lib).resolve()))
    out = f"/tmp/tbv_{Path(lib).stem}.npy"
    r = subprocess.run([sys.executable, __file__, "--one", cfgname, out], env=env,
                       capture_output=True, text=True)
    if r.returncode != 0:
        print(lib, "FAILED", r.stderr[-2000:])
        continue
    res = json.loads(r.stdout.strip().splitlines()[-1])
    g = np.load(out)
    if first is None:
        first = g
    res["maxrel_vs_first"] = float(np.abs(g - first).max() / max(np.abs(first).max(), 1e-30))
    print(Path(lib).name, json.dumps(res), flush=True)
