"""Per-phase warp-time breakdown of the forward kernel (experiment build).

    nvcc ... -DGSX_PHASE_PROF -shared -o paper_2509_07782_b200/libgsx_prof.so csrc/*.cu
    GSX_LIB=$PWD/paper_2509_07782_b200/libgsx_prof.so python profiles/phase_prof.py [c3|c1]
"""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_07782_b200 as G  # noqa: E402
from paper_2509_07782_b200 import _lib  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
variant = sys.argv[2] if len(sys.argv) > 2 else None
rec, eps, cam_kw, cfg_kw, desc = bench.workload(cfgname)
scene = G.Scene.from_records(rec)
G.reorder_by_morton(scene)
cam = bench.make_camera(G, cam_kw)
log = None
if len(sys.argv) > 3 and sys.argv[3] == "logged":  # the training forward
    from paper_2509_07782_b200.renderer import MarchLog
    log = MarchLog(cam)
cfg = G.RenderConfig(**cfg_kw)
L = _lib.lib()
L.gsx_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 24)()
for _ in range(2):
    G.render(scene, cam, cfg, variant=variant, log=log)
torch.cuda.synchronize()
L.gsx_phase_times(buf, 1)
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
G.render(scene, cam, cfg, variant=variant, log=log)
e1.record(s)
torch.cuda.synchronize()
L.gsx_phase_times(buf, 1)
names = ["closest_hit(initial)", "warp_traverse", "list_process", "composite",
         "phantom/stats | exact emptiness over the list (screened)", "advance(+ESS closest hit)",
         "march_total", "emptiness_tail (screened)"]
tot = buf[6] or 1
out = {n: {"warp_cycles": int(buf[i]), "share_of_march": buf[i] / tot} for i, n in enumerate(names)}
warps = (cam.width * cam.height + 31) // 32
counts = {"warp_node_steps": buf[8], "warp_list_entries": buf[9], "warp_iterations": buf[10],
          "lane_candidate_uses": buf[11], "lane_candidate_tests": buf[12], "reuses": buf[15],
          "active_lane_iterations": buf[13],
          "per_warp": {"node_steps": buf[8] / warps, "list_entries": buf[9] / warps,
                       "iterations": buf[10] / warps},
          "per_iteration": {"node_steps": buf[8] / max(buf[10], 1),
                            "list_entries": buf[9] / max(buf[10], 1),
                            "active_lanes": buf[13] / max(buf[10], 1)},
          "use_fraction": buf[11] / max(buf[12], 1),
          "entries_any_use_fraction": buf[14] / max(buf[9], 1),
          "lanes_per_used_entry": buf[11] / max(buf[14], 1),
          "cycles_per_node_step": buf[1] / max(buf[8], 1),
          "cycles_per_list_entry": buf[2] / max(buf[9], 1)}
screened = {"screen (per batch)": buf[16], "setup (per screened-in entry)": buf[17],
            "radiance (per used entry)": buf[18], "samples (per used entry)": buf[19]}
screened = {k: {"warp_cycles": int(v), "share_of_march": v / tot} for k, v in screened.items()}
counts["screened_in_entries"] = buf[21]
counts["used_entries"] = buf[20]
print(json.dumps({"config": cfgname, "ms": e0.elapsed_time(e1), "phases": out,
                  "screened_list": screened, "counts": counts}, indent=1))
