"""C5 sweep (BASELINE.json config 5): BVH build cost and
traversal cost versus scene size and anisotropy, with and without the
volume-ratio AABB bound (PAPER.md 1091-1092, geometry.py:193-212).

    python bench_c5.py [--sizes 100000,300000,...] [--aniso 1,10,100,1000]
                       [--width 480 --height 270] [--out profiles/c5_sweep.json]

Per run: the device rebuild (K1 prepare + bounds, K2 Morton, K3 sort, K5
LBVH + 4-wide collapse) timed with CUDA events (median of 5; eager launches
and the CUDA-graph replay), the forward render of one camera (adaptive + ESS,
median of 3, every forward variant timed and the fastest reported) in
Mrays/s, and
per-ray reference-semantics counters on a 4096-ray subset
(gsx_render_rays_stats): node visits, AABB hits, ellipsoid hits and the
false-positive fraction (bench.py:181-198).  Scenes: synth_records("ball")
with scales (b, b, a b), uniform random rotations; "bound" clamps a so that
ratio_upper_bound((1,1,a)) <= r0 = 10 (a <= 4.914).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent


def run_one(G, n, aniso, bound, width, height, seed=0):
    import torch

    from paper_2509_07782_b200.renderer import ray_stats
    from paper_2509_07782_b200.scenes import synth_records

    t0 = time.time()
    rec = synth_records("ball", n, seed=seed, anisotropy=aniso,
                        r_max_bound=10.0 if bound else None)
    gen_s = time.time() - t0
    scene = G.Scene.from_records(rec)
    G.reorder_by_morton(scene)
    s = torch.cuda.current_stream()

    def timed(fn, reps):
        fn()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    build_ms = timed(scene.rebuild_async, 5)
    build_graph_ms = timed(scene.rebuild_graphed, 5)
    cam = G.orbit_cameras(1, radius=3.5, focal=1.2 * width, width=width, height=height)[0]
    cfg = G.RenderConfig(mode="adaptive")
    from paper_2509_07782_b200.renderer import VARIANTS

    by_variant = {v: timed(lambda: G.render(scene, cam, cfg, variant=v), 3) for v in VARIANTS}
    best = min(by_variant, key=by_variant.get)
    ms = by_variant[best]
    # reference-semantics counters on a strided ray subset
    step = max(1, int(np.sqrt(width * height / 4096)))
    py, px = np.mgrid[0:height:step, 0:width:step]
    rays = cam.rays(np.stack([px.ravel(), py.ravel()], axis=1))
    per = ray_stats(scene, rays, cfg, clip=True).astype(np.float64)
    hit = per[:, 0] > 0
    aabb, ell = per[:, 6].sum(), per[:, 7].sum()
    a_eff = min(aniso, 4.914) if bound else aniso
    return {"n": n, "anisotropy": aniso, "bound": bound, "anisotropy_effective": a_eff,
            "gen_s": round(gen_s, 3), "build_ms": build_ms, "build_graph_ms": build_graph_ms,
            "render_ms": ms, "render_variant": best,
            "render_ms_by_variant": {k: round(v, 3) for k, v in by_variant.items()},
            "mrays_s": width * height / ms / 1e3,
            "node_visits_per_ray": float(per[hit, 5].mean()) if hit.any() else 0.0,
            "aabb_hits_per_ray": float(per[hit, 6].mean()) if hit.any() else 0.0,
            "ellipsoid_hits_per_ray": float(per[hit, 7].mean()) if hit.any() else 0.0,
            "false_positive_fraction": float((aabb - ell) / aabb) if aabb else 0.0,
            "samples_per_ray": float(per[hit, 1].mean()) if hit.any() else 0.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="100000,300000,1000000,3000000,5000000")
    ap.add_argument("--aniso", default="1,10,100,1000")
    ap.add_argument("--aniso-n", type=int, default=1_000_000)
    ap.add_argument("--width", type=int, default=480)
    ap.add_argument("--height", type=int, default=270)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    sys.path.insert(0, str(ROOT))
    import paper_2509_07782_b200 as G

    rows = []
    for n in [int(x) for x in args.sizes.split(",") if x]:
        rows.append(run_one(G, n, 1.0, False, args.width, args.height))
        print(json.dumps(rows[-1]), flush=True)
    for a in [float(x) for x in args.aniso.split(",") if x]:
        for bound in (False, True):
            rows.append(run_one(G, args.aniso_n, a, bound, args.width, args.height))
            print(json.dumps(rows[-1]), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps({"config": "C5 sweep", "width": args.width,
                                              "height": args.height, "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
