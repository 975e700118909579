"""One training step of the RayGaussX objective on the B200 kernels.

The reference has no training loop (pkg/README.md:137-138; its only gradient
is a finite-difference oracle, densify.py:156-187).  This module composes the
render path into the step BASELINE.json configs C2 / C4 time:

    K1-K5 rebuild (prepare, Morton, radix sort, LBVH; the BVH is rebuilt every
    step)  ->  forward on this rank's 16x16 tiles  ->  tile
    assembly (NCCL all-reduce of disjoint tiles)  ->  L1 + DSSIM loss and
    dL/dI on the full frame (K8)  ->  backward on this rank's tiles (K7)  ->
    isotropic-loss gradient (K9, rank 0)  ->  NCCL all-reduce of the [N,87]
    gradient  ->  fused Adam with projection onto valid records.

Rays shard across GPUs by tile (tile t -> rank t mod G); every rank holds the
full parameter set and builds its own (deterministic, identical) BVH.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr, stream_ptr
from .config import Camera, RenderConfig
from .loss import ImageLoss, IsoLossConfig, LossConfig
from .renderer import MarchLog, render, render_backward

# default per-slot learning rates of the 87-float record
LR_GROUPS = {"mean": (0, 3, 1e-4), "quat": (3, 7, 1e-3), "scale": (7, 10, 1e-4),
             "sigma": (10, 11, 5e-2), "sh": (11, 38, 2.5e-3), "axis": (38, 59, 1e-3),
             "sharp": (59, 66, 1e-2), "amp": (66, 87, 2.5e-3)}


TILE_ORDER = 1  # GSX_TILE_ORDER (csrc/gsx_common.cuh)


def tile_at(s: int, tiles_x: int, tiles_y: int, stride: int) -> int:
    """Row-major tile id at tile-sequence position s of a launch with
    tile_stride `stride`: for stride > 1 the tile rows run centre-out
    (c, c+1, c-1, ...; c = (tiles_y-1)//2) -- gsx_tile_at, csrc/gsx_common.cuh."""
    if not TILE_ORDER or stride <= 1:
        return s
    i, c = s // tiles_x, (tiles_y - 1) // 2
    d = (i + 1) // 2
    row = c + d if i & 1 else c - d
    return row * tiles_x + s % tiles_x


def tiles_of_rank(n_tiles: int, rank: int, world: int, tiles_x: int | None = None) -> list:
    """Row-major tile ids rendered by `rank` (tile_begin=rank,
    tile_stride=world): sequence positions rank + k*world (interleaved for
    load balance), through the centre-out row order when world > 1.  tiles_x = tiles per
    image row (default: n_tiles, i.e. one row)."""
    tx = n_tiles if tiles_x is None else tiles_x
    ty = n_tiles // tx
    return [tile_at(s, tx, ty, world) for s in range(rank, n_tiles, world)]


def assemble_tiles(buffers, group=None):
    """Sum disjoint per-rank tile buffers (zero outside the rank's tiles) into
    the full frame on every rank (one all-reduce over the concatenation)."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return buffers
    flat = torch.cat([b.reshape(-1) for b in buffers])
    dist.all_reduce(flat, group=group)
    out, off = [], 0
    for b in buffers:
        b.copy_(flat[off:off + b.numel()].view_as(b))
        off += b.numel()
        out.append(b)
    return out


def allreduce_grad(grad, group=None):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad, group=group)
    return grad


class Adam:
    """Fused Adam over [N,87] records (gsx_adam_step) with per-slot learning
    rates and a projection keeping every record valid (sigma~ > sigma_eps,
    scales >= 1e-7, sharpness >= 0)."""

    def __init__(self, params, sigma_eps: float, lr=None, betas=(0.9, 0.999), eps=1e-15):
        dev = params.device
        self.params = params
        self.m = torch.zeros_like(params)
        self.v = torch.zeros_like(params)
        lr87 = np.zeros(87, np.float32)
        for name, (a, b, default) in LR_GROUPS.items():
            lr87[a:b] = (lr or {}).get(name, default)
        lo87 = np.full(87, -np.inf, np.float32)
        lo87[10] = np.float32(sigma_eps * 1.0001)
        lo87[7:10] = 1e-7
        lo87[59:66] = 0.0
        self.lr87 = torch.as_tensor(lr87, device=dev)
        self.lo87 = torch.as_tensor(lo87, device=dev)
        self.betas, self.eps, self.t = betas, eps, 0

    def step(self, grad):
        self.t += 1
        L = _lib.lib()
        check(L.gsx_adam_step(ptr(self.params), ptr(grad), ptr(self.m), ptr(self.v),
                              self.params.shape[0], ptr(self.lr87), ptr(self.lo87),
                              float(self.betas[0]), float(self.betas[1]), float(self.eps),
                              self.t, stream_ptr()), "adam")


class Trainer:
    """Stateful train step for one scene (`scene.params` are optimized in place)."""

    def __init__(self, scene, camera: Camera, cfg: RenderConfig | None = None,
                 loss_cfg: LossConfig = LossConfig(), iso_cfg: IsoLossConfig = IsoLossConfig(),
                 lr=None, group=None, march_log: bool = True, densify=None):
        import torch.distributed as dist

        self.scene, self.camera = scene, camera
        self.cfg = cfg or RenderConfig()
        self.loss_cfg, self.iso_cfg = loss_cfg, iso_cfg
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        H, W = camera.height, camera.width
        dev = scene.device
        self.rgb = torch.zeros((H, W, 3), device=dev)
        self.depth = torch.zeros((H, W), device=dev)
        self.trans = torch.zeros((H, W), device=dev)
        self.dI = torch.empty((H, W, 3), device=dev)
        self.grad = torch.zeros_like(scene.params)
        self.loss = ImageLoss(H, W, 3, dev)
        self.adam = Adam(scene.params, scene.sigma_eps, lr)
        self._iso = torch.zeros(1, dtype=torch.float64, device=dev)
        # the forward records its march for the backward (renderer.MarchLog)
        self.log = (MarchLog(camera, tile_begin=self.rank, tile_stride=self.world, device=dev)
                    if march_log else None)
        self._steps = 0
        # optional densify.GradAccumulator observing every step's view
        self.densify = densify

    def step(self, target, want_loss: bool = False):
        """One optimization step against `target` [H,W,3] (CUDA).  Returns the
        loss value (host sync) when want_loss, else None."""
        s = self.scene
        L = _lib.lib()
        s.rebuild_async()
        if self.world > 1:
            self.rgb.zero_()
            self.depth.zero_()
            self.trans.zero_()
        render(s, self.camera, self.cfg, tile_begin=self.rank, tile_stride=self.world,
               rgb=self.rgb, depth=self.depth, trans=self.trans, log=self.log)
        assemble_tiles([self.rgb, self.depth, self.trans], self.group)
        vals, _ = self.loss(self.rgb, target, self.loss_cfg.mix, grad=self.dI,
                            want_value=want_loss)
        self.grad.zero_()
        render_backward(s, self.camera, self.cfg, self.rgb, self.depth, self.trans, self.dI,
                        grad=self.grad, tile_begin=self.rank, tile_stride=self.world,
                        log=self.log)
        if self.rank == 0 and self.iso_cfg.lambda_s > 0:
            check(L.gsx_iso_loss(ptr(s.params), s.n, float(self.iso_cfg.r0),
                                 float(self.iso_cfg.lambda_s), ptr(self.grad), ptr(self._iso),
                                 stream_ptr()), "iso_loss")
        allreduce_grad(self.grad, self.group)
        if self.densify is not None:  # |dL/dmu| of this view, before the update
            self.densify.observe_view(self.grad, s.params, self.camera)
        self.adam.step(self.grad)
        self._steps += 1
        if self.log is not None and (self._steps == 1 or want_loss):
            self.log.ensure()  # overflowed warps were replayed; size up for the next step
        if want_loss:
            iso = float(self._iso.item()) / s.n if self.rank == 0 else 0.0
            return vals[0] + self.iso_cfg.lambda_s * iso
        return None
