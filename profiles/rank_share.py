"""Per-rank share of the C3 forward, timed alone on one GPU.

    python profiles/rank_share.py [--worlds 2,4,8] [--reps 5] [--out FILE]

Under `bench.py --gpus N` rank r renders the 16x16 tiles r, r+N, r+2N, ...
(tile_begin=r, tile_stride=N) and the frame is assembled by one all-gather.
Each rank's render is independent of the others (no data-path collective), so
its device time can be measured on one GPU by launching exactly that rank's
share: the same kernel, grid and tiles the rank launches.  For every N this
prints the per-rank median ms (L2 flushed before each launch, CUDA events on
the launching stream), max over ranks, and the forward-only scaling
efficiency t_1 / (N * max_r t_r) the render kernel allows (the all-gather of
the 41 MB rgb+depth+T frame is not included).  Each world reports the best of
the forward variants (the library autotunes per tile-set shape).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--variants", default="screened,screened-regs,plain",
                    help="forward variants to time (renderer.VARIANTS); each world "
                         "reports its best")
    args = ap.parse_args()

    import torch

    import bench
    import paper_2509_07782_b200 as G

    rec, eps, cam_kw, cfg_kw, desc = bench.workload("c3")
    dev = torch.device("cuda", 0)
    scene = G.Scene.from_records(torch.from_numpy(rec.astype("float32")).to(dev))
    G.reorder_by_morton(scene)
    cam = bench.make_camera(G, cam_kw)
    cfg = G.RenderConfig(**cfg_kw)
    H, W = cam_kw["height"], cam_kw["width"]
    rgb = torch.zeros((H, W, 3), device=dev)
    depth = torch.zeros((H, W), device=dev)
    trans = torch.zeros((H, W), device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream()

    def time_share(tb, ts, variant):
        for _ in range(2):
            G.render(scene, cam, cfg, tile_begin=tb, tile_stride=ts, rgb=rgb, depth=depth,
                     trans=trans, variant=variant)
        ms = []
        for _ in range(args.reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            G.render(scene, cam, cfg, tile_begin=tb, tile_stride=ts, rgb=rgb, depth=depth,
                     trans=trans, variant=variant)
            b.record(s)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        return sorted(ms)[len(ms) // 2]

    variants = args.variants.split(",")
    t1s = {v: time_share(0, 1, v) for v in variants}
    v1 = min(t1s, key=t1s.get)
    t1 = t1s[v1]
    out = {"workload": desc, "t1_ms": t1, "t1_variant": v1, "t1_by_variant": t1s, "worlds": []}
    for n in [int(x) for x in args.worlds.split(",")]:
        best = None
        for v in variants:
            per = [time_share(r, n, v) for r in range(n)]
            mx = max(per)
            row = {"n": n, "variant": v, "per_rank_ms": per, "max_ms": mx, "sum_ms": sum(per),
                   "forward_efficiency": t1 / (n * mx)}
            print(json.dumps(row), flush=True)
            if best is None or mx < best["max_ms"]:
                best = row
        out["worlds"].append(best)
    print(json.dumps({"t1_ms": t1, "t1_variant": v1}), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
