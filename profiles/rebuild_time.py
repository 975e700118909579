"""Device ms of one K1-K5 rebuild (eager and CUDA-graph replay) for the
workloads given, and the per-kernel split when run under ncu's launch list.

    python profiles/rebuild_time.py c3 c4
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_07782_b200 as G  # noqa: E402

for name in sys.argv[1:] or ["c4"]:
    rec, eps, cam_kw, cfg_kw, desc = bench.workload(name)
    scene = G.Scene.from_records(rec)
    G.reorder_by_morton(scene)
    s = torch.cuda.current_stream()
    out = {"config": name, "n": int(rec.shape[0])}
    for label, fn in (("eager", scene.rebuild_async), ("graph", scene.rebuild_graphed)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(10):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        out[label + "_ms"] = e0.elapsed_time(e1) / 10
    print(json.dumps(out), flush=True)
    del scene
    torch.cuda.empty_cache()
