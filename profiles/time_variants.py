"""Time the forward render of one workload for several libgsx builds (experiment
variants compiled with different -D flags), in one process per variant:

    python profiles/time_variants.py c3 lib_a.so lib_b.so ...

Prints one line per variant: median ms over 7 renders after 2 warm-ups
(L2 flushed before each) and the max |rgb - first variant's rgb|.
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
    rec, eps, cam_kw, cfg_kw, desc = bench.workload(cfgname)
    scene = G.Scene.from_records(rec)
    G.reorder_by_morton(scene)
    cam = bench.make_camera(G, cam_kw)
    cfg = G.RenderConfig(**cfg_kw)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(9):
        flush.zero_()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        rgb, _, _, _ = G.render(scene, cam, cfg)
        e1.record(s)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    np.save(out, rgb.cpu().numpy())
    print(json.dumps({"ms": float(np.median(ts)), "min": float(min(ts))}))
    sys.exit(0)

cfgname, libs = sys.argv[1], sys.argv[2:]
import numpy as np  # noqa: E402
first = None
for lib in libs:
    env = dict(os.environ, GSX_LIB=str(Path(lib).resolve()))
    out = f"/tmp/tv_{Path(lib).stem}.npy"
    r = subprocess.run([sys.executable, __file__, "--one", cfgname, out], env=env,
                       capture_output=True, text=True)
    if r.returncode != 0:
        print(lib, "FAILED", r.stderr[-2000:])
        continue
    res = json.loads(r.stdout.strip().splitlines()[-1])
    img = np.load(out)
    if first is None:
        first = img
    res["maxdiff_vs_first"] = float(np.abs(img - first).max())
    print(Path(lib).name, json.dumps(res), flush=True)
