"""Multi-process (gloo, world 2 and 4, CPU) tests of the tile-sharded
training-step orchestration in paper_2509_07782_b200/train.py:

* tile ownership (`tiles_of_rank`, the library's own tile order gsx_tile_id);
* frame assembly by an all-gather of each rank's own tiles (`gather_tiles`);
* the ZeRO-1 style update (`sharded_update`): reduce-scatter of the [N,87]
  gradient into row shards, the optimizer on this rank's shard, all-gather
  of the parameter shards.

The per-tile render / backward is the float64 oracle here (no GPU) and the
optimizer a plain SGD step standing in for gsx_adam_step, so the sharded
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

H, W = 40, 56  # 4 x 3 tiles, ragged in both directions
LR = 0.05


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
    from paper_2509_07782_b200.train import gather_tiles, shard_rows, sharded_update, tiles_of_rank

    rec, rays, target = _setup()
    osc = O.OracleScene(rec)
    cfg = O.OCfg.make(dt=0.01)
    tx, ty = (W + 15) // 16, (H + 15) // 16
    mine = [p for t in tiles_of_rank(tx, ty, rank, world) for p in _tile_pixels(t)]
    # garbage outside this rank's tiles: the gather must overwrite every pixel
    rgb = torch.full((H, W, 3), np.nan, dtype=torch.float64)
    depth = torch.full((H, W), np.nan, dtype=torch.float64)
    trans = torch.full((H, W), np.nan, dtype=torch.float64)
    r = np.array([rays[y, x] for y, x in mine])
    R, T, D, _ = osc.march_rays(r, cfg)
    for (y, x), c, tt, dd in zip(mine, R, T, D):
        rgb[y, x] = torch.as_tensor(c)
        trans[y, x] = tt
        depth[y, x] = dd
    gather_tiles([rgb, depth, trans], W, H)
    gI = OL.image_loss_grad(rgb.numpy(), target, 0.2)
    gC = np.array([gI[y, x] for y, x in mine])
    _, _, _, grad = osc.backward_rays(r, cfg, gC, np.zeros(len(mine)), np.zeros(len(mine)))
    n = rec.shape[0]
    rows = shard_rows(n, world)
    gpad = torch.zeros((rows * world, 87), dtype=torch.float64)
    gpad[:n] = torch.as_tensor(grad)
    ppad = torch.zeros((rows * world, 87), dtype=torch.float64)
    ppad[:n] = torch.as_tensor(rec.astype(np.float64))

    def sgd(p, g):
        p.sub_(LR * g)

    sharded_update(gpad, ppad, sgd)
    return (rgb.numpy(), depth.numpy(), trans.numpy()), ppad[:n].numpy()


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frame, p = _step(rank, world)
        np.save(os.path.join(out, f"rgb{rank}.npy"), frame[0])
        np.save(os.path.join(out, f"depth{rank}.npy"), frame[1])
        np.save(os.path.join(out, f"p{rank}.npy"), p)
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
            per = [tiles_of_rank(tx, ty, r, world) for r in range(world)]
            seen = sorted(t for p in per for t in p)
            assert seen == list(range(n_tiles)), (tx, ty, world)
    # sharded launches visit the tile rows centre-out; a whole image is row-major
    assert tiles_of_rank(120, 68, 0, 2)[:2] == [33 * 120, 33 * 120 + 2]
    assert tiles_of_rank(120, 68, 0, 1)[:2] == [0, 1]
    with pytest.raises(ValueError):
        from paper_2509_07782_b200.train import tile_at
        tile_at(35, 7, 5, 2)


def test_rank_pixels_cover_frame():
    from paper_2509_07782_b200.train import rank_pixels

    for world in (1, 2, 3, 4, 8):
        pix = rank_pixels(W, H, world, "cpu").numpy()
        got = np.sort(pix[pix >= 0])
        assert np.array_equal(got, np.arange(W * H)), world


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_step_equals_single_process(tmp_path, world):
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    (rgb1, depth1, _), p1 = _step(0, 1)
    rec = _setup()[0]
    assert np.abs(p1 - rec).max() > 0  # the step moved the parameters
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"rgb{r}.npy"), rgb1)
        np.testing.assert_array_equal(np.load(tmp_path / f"depth{r}.npy"), depth1)
        p = np.load(tmp_path / f"p{r}.npy")
        np.testing.assert_allclose(p, p1, rtol=1e-12, atol=1e-12 * np.abs(p1).max())
