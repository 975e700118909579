"""Per-phase warp-time breakdown of the logged backward's pair path
(experiment build with -DGSX_PHASE_PROF, profiles/build_prof.sh):

    GSX_LIB=$PWD/paper_2509_07782_b200/libgsx_prof.so python profiles/phase_prof_bwd.py c4 [pass2]
"""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_07782_b200 as G  # noqa: E402
from paper_2509_07782_b200 import _lib  # noqa: E402
from paper_2509_07782_b200.renderer import MarchLog  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c4"
pass2 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rec, eps, cam_kw, cfg_kw, desc = bench.workload(cfgname)
scene = G.Scene.from_records(rec)
G.reorder_by_morton(scene)
cam = bench.make_camera(G, cam_kw)
cfg = G.RenderConfig(**cfg_kw)
L = _lib.lib()
L.gsx_phase_times_bwd.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 24)()
log = MarchLog(cam)
for _ in range(2):
    G.render(scene, cam, cfg, log=log)
    log.ensure()
rgb, depth, trans, _ = G.render(scene, cam, cfg, log=log)
g = torch.randn_like(rgb) * 1e-3
G.render_backward(scene, cam, cfg, rgb, depth, trans, g, log=log, pass2=pass2)
torch.cuda.synchronize()
L.gsx_phase_times_bwd(buf, 1)
G.render_backward(scene, cam, cfg, rgb, depth, trans, g, log=log, pass2=pass2)
torch.cuda.synchronize()
L.gsx_phase_times_bwd(buf, 1)
names = ["record prologue (adjoints)", "pair setup", "radiance", "moments",
         "P1 columns + reduce", "P2/P3 lobes + reduce", "batch flush"]
tot = sum(buf[i] for i in range(7)) or 1
sub = {"P2/P3 lobe columns": buf[10], "P2/P3 reduce + emit": buf[11]}
print(json.dumps({"config": cfgname, "pass2": pass2, "batches": buf[9],
                  "p23_split": {k: v / tot for k, v in sub.items()},
                  "phases": {n: {"warp_cycles": int(buf[i]), "share": buf[i] / tot}
                             for i, n in enumerate(names)}}, indent=1))
