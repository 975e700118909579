"""Multi-process (gloo, world_size 2, CPU) test of the tile-sharded training-step
orchestration in paper_2509_07782_b200/train.py: tile ownership, tile
assembly (all-reduce of disjoint tiles) and the gradient all-reduce.  The
per-tile render/backward is the float64 oracle here (no GPU), so the sharded
result must equal the single-process full-frame result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from oracle import loss as OL
from paper_2509_07782_b200.scenes import f32_records, gen_test_scene_records, orbit_poses

H, W = 32, 48


def _setup():
    rec = f32_records(gen_test_scene_records("random-cloud", count=40, seed=2, anisotropy=2.0,
                                             base_scale=0.12))
    center, quat = orbit_poses(1, 3.0)[0]
    rays = O.camera_rays(center, quat, 30.0, W, H).reshape(H, W, 8)
    target = np.random.default_rng(0).uniform(0, 0.5, size=(H, W, 3))
    return rec, rays, target


def _tile_pixels(t):
    tiles_x = (W + 15) // 16
    ty, tx = divmod(t, tiles_x)
    return [(y, x) for y in range(16 * ty, min(16 * ty + 16, H))
            for x in range(16 * tx, min(16 * tx + 16, W))]


def _step(rank, world):
    from paper_2509_07782_b200.train import allreduce_grad, assemble_tiles, tiles_of_rank

    rec, rays, target = _setup()
    osc = O.OracleScene(rec)
    cfg = O.OCfg.make(dt=0.01)
    n_tiles = ((W + 15) // 16) * ((H + 15) // 16)
    mine = [p for t in tiles_of_rank(n_tiles, rank, world) for p in _tile_pixels(t)]
    rgb = torch.zeros((H, W, 3), dtype=torch.float64)
    depth = torch.zeros((H, W), dtype=torch.float64)
    trans = torch.zeros((H, W), dtype=torch.float64)
    r = np.array([rays[y, x] for y, x in mine])
    R, T, D, _ = osc.march_rays(r, cfg)
    for (y, x), c, tt, dd in zip(mine, R, T, D):
        rgb[y, x] = torch.as_tensor(c)
        trans[y, x] = tt
        depth[y, x] = dd
    assemble_tiles([rgb, depth, trans])
    gI = OL.image_loss_grad(rgb.numpy(), target, 0.2)
    gC = np.array([gI[y, x] for y, x in mine])
    _, _, _, grad = osc.backward_rays(r, cfg, gC, np.zeros(len(mine)), np.zeros(len(mine)))
    g = torch.as_tensor(grad)
    allreduce_grad(g)
    return rgb.numpy(), g.numpy()


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rgb, g = _step(rank, world)
        np.save(os.path.join(out, f"rgb{rank}.npy"), rgb)
        np.save(os.path.join(out, f"g{rank}.npy"), g)
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_tiles_partition():
    from paper_2509_07782_b200.train import tiles_of_rank

    for tx, ty in ((1, 1), (7, 1), (7, 5), (10, 10), (79, 51), (120, 68), (120, 67)):
        n_tiles = tx * ty
        for world in (1, 2, 3, 5, 8):
            per = [tiles_of_rank(n_tiles, r, world, tx) for r in range(world)]
            seen = sorted(t for p in per for t in p)
            assert seen == list(range(n_tiles)), (tx, ty, world)
    # sharded launches visit the tile rows centre-out; a whole image is row-major
    assert tiles_of_rank(8160, 0, 2, 120)[:2] == [33 * 120, 33 * 120 + 2]
    assert tiles_of_rank(8160, 0, 1, 120)[:2] == [0, 1]


@pytest.mark.parametrize("world", [2])
def test_sharded_step_equals_single_process(tmp_path, world):
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    rgb1, g1 = _step(0, 1)
    for r in range(world):
        rgb = np.load(tmp_path / f"rgb{r}.npy")
        g = np.load(tmp_path / f"g{r}.npy")
        np.testing.assert_allclose(rgb, rgb1, rtol=0, atol=1e-15)
        np.testing.assert_allclose(g, g1, rtol=1e-12, atol=1e-12 * np.abs(g1).max())
