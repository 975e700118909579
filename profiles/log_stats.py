"""Pair statistics of a training forward's march log (march_log.cuh layout):
list entries, (lane, primitive) pairs from the use masks, and how the logged
backward's pass 2 batches them (32 pairs per batch, per record list, per
group of 32 entries).   python profiles/log_stats.py c2|c4"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_07782_b200 as G  # noqa: E402
from paper_2509_07782_b200.renderer import MarchLog, render  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
rec, eps, cam_kw, cfg_kw, desc = bench.workload(cfgname)
cam = bench.make_camera(G, cam_kw)
cfg = G.RenderConfig(**cfg_kw)
scene = G.Scene.from_records(rec)
G.reorder_by_morton(scene)
log = MarchLog(cam)
render(scene, cam, cfg, log=log)
used, ovf = log.usage()
torch.cuda.synchronize()
head = int(log.arena[:8].view(torch.int64).item())
buf = log.arena[:head].cpu().numpy()
off = log.min_bytes


def r128(x):
    return (x + 127) & ~127


def r16(x):
    return (x + 15) & ~15


popc = np.array([bin(i).count("1") for i in range(256)], dtype=np.int64)
n_rec = [0, 0]
entries = pairs = batches = runs = groups = 0
hist = np.zeros(33, dtype=np.int64)
while off < head:
    h = buf[off:off + 32]
    cnt = int(h[8:12].view(np.int32)[0])
    kind = int(h[12:16].view(np.int32)[0])
    mmax = int(h[16:20].view(np.int32)[0])
    act = int(h[20:24].view(np.uint32)[0])
    cap = int(h[24:28].view(np.int32)[0])
    sw = int(h[28:32].view(np.int32)[0])
    body = off + 128
    if kind == 1:
        lst, um = body, body + r16(4 * cap)
        size = 128 + r128(r16(4 * cap) + 4 * cap)
    else:
        nact = bin(act).count("1")
        smp = r16(20 * nact)
        lo = smp + 16 * (sw or nact) * mmax
        lst, um = body + lo, body + lo + r16(4 * cap)
        size = 128 + r128(lo + r16(4 * cap) + 4 * cap)
    n_rec[kind] += 1
    m = buf[um:um + 4 * cnt].view(np.uint32).astype(np.int64)
    pc = popc[m & 255] + popc[(m >> 8) & 255] + popc[(m >> 16) & 255] + popc[m >> 24]
    hist += np.bincount(pc, minlength=33)
    entries += cnt
    pairs += int(pc.sum())
    for g0 in range(0, cnt, 32):
        gp = pc[g0:g0 + 32]
        tot = int(gp.sum())
        groups += 1
        nb = (tot + 31) // 32
        batches += nb
        # runs: entries per batch, +1 for each entry split by a batch boundary
        ends = np.cumsum(gp)
        runs += int((gp > 0).sum()) + sum(int(((ends > 32 * b) & (ends - gp < 32 * b)).sum())
                                          for b in range(1, nb))
    off += size
out = {"config": cfgname, "log_bytes": head, "overflow": ovf, "records_full": n_rec[0],
       "records_list": n_rec[1], "entries": entries, "pairs": pairs,
       "pairs_per_entry": pairs / max(entries, 1), "groups": groups, "batches": batches,
       "pairs_per_batch": pairs / max(batches, 1), "runs_per_batch": runs / max(batches, 1),
       "entries_per_full_record": entries / max(n_rec[0], 1),
       "popc_hist": hist.tolist()}
print(json.dumps(out))
