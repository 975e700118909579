"""One training step of the RayGaussX objective on the B200 kernels.

The reference has no training loop (pkg/README.md:137-138; its only gradient
is a finite-difference oracle, densify.py:156-187).  This module composes the
render path into the step BASELINE.json configs C2 / C4 time:

    K1-K5 rebuild (prepare, Morton, radix sort, LBVH; the BVH is rebuilt every
    step)  ->  forward on this rank's 16x16 tiles  ->  tile
    assembly (NCCL all-gather of the ranks' own tiles)  ->  L1 + DSSIM loss
    and dL/dI on the full frame (K8)  ->  backward on this rank's tiles (K7)
    ->  isotropic-loss gradient (K9, rank 0)  ->  NCCL reduce-scatter of the
    [N,87] gradient into row shards  ->  fused Adam with projection onto
    valid records on this rank's shard  ->  NCCL all-gather of the shards.

Rays shard across GPUs by tile (tile t -> rank t mod G); every rank holds the
full parameter set and builds its own (deterministic, identical) BVH.
"""

from __future__ import annotations

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


def tile_at(s: int, tiles_x: int, tiles_y: int, stride: int) -> int:
    """Row-major tile id at tile-sequence position s of a launch with
    tile_stride `stride` -- asked of the library (gsx_tile_id, the kernels'
    own gsx_tile_at), so the host cannot drift from the device order."""
    t = int(_lib.load_library().gsx_tile_id(int(s), int(tiles_x), int(tiles_y), int(stride)))
    if t < 0:
        raise ValueError(f"tile position {s} outside a {tiles_x}x{tiles_y} grid")
    return t


def tiles_of_rank(tiles_x: int, tiles_y: int, rank: int, world: int) -> list:
    """Row-major tile ids rendered by `rank` (tile_begin=rank,
    tile_stride=world): sequence positions rank + k*world (interleaved for
    load balance), through the library's tile order (centre-out rows when
    world > 1)."""
    n = int(tiles_x) * int(tiles_y)
    return [tile_at(s, tiles_x, tiles_y, world) for s in range(rank, n, world)]


_PIX_CACHE: dict = {}


def rank_pixels(width: int, height: int, world: int, device):
    """Flat pixel indices (py * width + px) of every rank's tiles, padded to
    one length with -1: LongTensor [world, P], cached per (W, H, world)."""
    key = (int(width), int(height), int(world), str(device))
    if key not in _PIX_CACHE:
        tx, ty = (width + 15) // 16, (height + 15) // 16
        rows = []
        for r in range(world):
            idx = []
            for t in tiles_of_rank(tx, ty, r, world):
                y0, x0 = 16 * (t // tx), 16 * (t % tx)
                ys = np.arange(y0, min(y0 + 16, height))
                xs = np.arange(x0, min(x0 + 16, width))
                idx.append((ys[:, None] * width + xs[None, :]).ravel())
            rows.append(np.concatenate(idx) if idx else np.zeros(0, np.int64))
        p = max(len(r) for r in rows)
        out = np.full((world, p), -1, np.int64)
        for r, row in enumerate(rows):
            out[r, :len(row)] = row
        _PIX_CACHE[key] = torch.as_tensor(out, device=device)
    return _PIX_CACHE[key]


def gather_tiles(buffers, width: int, height: int, group=None):
    """Assemble the full frame on every rank from the ranks' own tiles: each
    rank packs the pixels of its tiles ([H,W,C] or [H,W] buffers, channels
    concatenated), one all-gather moves the packed blocks, and every rank
    scatters them into place.  Moves one frame in total instead of an
    all-reduce over zero-padded full frames."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return buffers
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = buffers[0].device
    pix = rank_pixels(width, height, world, dev)
    flat = [b.reshape(width * height, -1) for b in buffers]
    widths = [f.shape[1] for f in flat]
    mine = pix[rank]
    valid = mine >= 0
    packed = torch.zeros((pix.shape[1], sum(widths)), dtype=buffers[0].dtype, device=dev)
    packed[valid] = torch.cat([f[mine[valid]] for f in flat], dim=1)
    allp = torch.empty((world * packed.shape[0], packed.shape[1]), dtype=packed.dtype,
                       device=dev)
    dist.all_gather_into_tensor(allp, packed, group=group)
    sel = pix.reshape(-1) >= 0
    rows = allp[sel]
    dst = pix.reshape(-1)[sel]
    off = 0
    for f, w in zip(flat, widths):
        f[dst] = rows[:, off:off + w]
        off += w
    return buffers


def assemble_tiles(buffers, group=None):
    """Sum disjoint per-rank tile buffers (zero outside the rank's tiles) into
    the full frame on every rank (one all-reduce over the concatenation).
    Kept for callers that render into zeroed buffers; `gather_tiles` moves
    only the owned tiles."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return buffers
    flat = torch.cat([b.reshape(-1) for b in buffers])
    dist.all_reduce(flat, group=group)
    off = 0
    for b in buffers:
        b.copy_(flat[off:off + b.numel()].view_as(b))
        off += b.numel()
    return buffers


def allreduce_grad(grad, group=None):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad, group=group)
    return grad


def shard_rows(n: int, world: int) -> int:
    """Rows per rank of the [N,87] parameter / gradient shards (N padded up
    to world * rows)."""
    return (int(n) + world - 1) // world


def sharded_update(grad_pad, params_pad, step_fn, group=None, reduced: bool = False,
                   gshard=None):
    """ZeRO-1-style update of row-padded [world*rows, 87] buffers: the summed
    gradient rows of this rank (reduce-scatter, or a slice when `grad_pad`
    is already all-reduced) -> step_fn(param_shard, grad_shard) updates this
    rank's parameter rows in place -> all-gather of the parameter shards."""
    import torch.distributed as dist

    on = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    if not on:
        step_fn(params_pad, grad_pad)
        return params_pad
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    rows = grad_pad.shape[0] // world
    lo = rank * rows
    if gshard is None:
        gshard = torch.empty((rows,) + tuple(grad_pad.shape[1:]), dtype=grad_pad.dtype,
                             device=grad_pad.device)
    if reduced:
        gshard.copy_(grad_pad[lo:lo + rows])
    else:
        dist.reduce_scatter_tensor(gshard, grad_pad, group=group)
    step_fn(params_pad[lo:lo + rows], gshard)
    dist.all_gather_into_tensor(params_pad, params_pad[lo:lo + rows].clone(), group=group)
    return params_pad


class Adam:
    """Fused Adam over [N,87] records (gsx_adam_step) with per-slot learning
    rates and a projection keeping every record valid (sigma~ > sigma_eps,
    scales >= 1e-7, sharpness >= 0).  `params` may be one rank's row shard
    (sharded optimizer state: m and v exist for those rows only)."""

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
    """Stateful train step for one scene (`scene.params` are optimized in place).

    With a process group of G > 1 ranks: every rank renders and back-propagates
    its own tiles; the frame is assembled by an all-gather of the owned tiles;
    the [N,87] gradient is reduce-scattered into G row shards, each rank runs
    Adam on its shard only (sharded m / v state), and an all-gather of the
    updated parameter shards gives every rank the full parameters for the
    next rebuild.  Same bytes on the wire as one all-reduce of the gradient,
    1/G of the optimizer work and state per rank."""

    def __init__(self, scene, camera: Camera, cfg: RenderConfig | None = None,
                 loss_cfg: LossConfig = LossConfig(), iso_cfg: IsoLossConfig = IsoLossConfig(),
                 lr=None, group=None, march_log: bool = True, densify=None,
                 graph_rebuild: bool = True):
        import torch.distributed as dist

        self.scene, self.camera = scene, camera
        self.graph_rebuild = graph_rebuild  # K1-K5 replayed as one CUDA graph
        self.cfg = cfg or RenderConfig()
        self.loss_cfg, self.iso_cfg = loss_cfg, iso_cfg
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        H, W = camera.height, camera.width
        dev = scene.device
        n = scene.n
        self.rows = shard_rows(n, self.world)
        npad = self.rows * self.world
        if self.world > 1:
            # parameters live in a row-padded buffer so the shards are equal
            # (scene.params stays the [N,87] view the kernels read)
            pad = torch.zeros((npad, 87), dtype=scene.params.dtype, device=dev)
            pad[:n] = scene.params
            scene.params = pad[:n]
            self._params_pad = pad
        self.rgb = torch.zeros((H, W, 3), device=dev)
        self.depth = torch.zeros((H, W), device=dev)
        self.trans = torch.zeros((H, W), device=dev)
        self.dI = torch.empty((H, W, 3), device=dev)
        self._grad_pad = torch.zeros((npad, 87), dtype=scene.params.dtype, device=dev)
        self.grad = self._grad_pad[:n]
        self.loss = ImageLoss(H, W, 3, dev)
        if self.world > 1:
            lo = self.rank * self.rows
            self._gshard = torch.empty((self.rows, 87), dtype=scene.params.dtype, device=dev)
            self.adam = Adam(self._params_pad[lo:lo + self.rows], scene.sigma_eps, lr)
        else:
            self.adam = Adam(scene.params, scene.sigma_eps, lr)
        self._iso = torch.zeros(1, dtype=torch.float64, device=dev)
        # the forward records its march for the backward (renderer.MarchLog)
        self.log = (MarchLog(camera, tile_begin=self.rank, tile_stride=self.world, device=dev)
                    if march_log else None)
        self._steps = 0
        # optional densify.GradAccumulator observing every step's view
        self.densify = densify

    def _optimizer_step(self, reduced: bool = False):
        """Adam over this rank's rows (all of them for one rank); see
        sharded_update."""
        if self.world == 1:
            self.adam.step(self.grad)
            return
        sharded_update(self._grad_pad, self._params_pad, lambda p, g: self.adam.step(g),
                       self.group, reduced, self._gshard)

    def step(self, target, want_loss: bool = False):
        """One optimization step against `target` [H,W,3] (CUDA).  Returns the
        loss value (host sync) when want_loss, else None."""
        s = self.scene
        L = _lib.lib()
        s.rebuild_graphed() if self.graph_rebuild else s.rebuild_async()
        render(s, self.camera, self.cfg, tile_begin=self.rank, tile_stride=self.world,
               rgb=self.rgb, depth=self.depth, trans=self.trans, log=self.log)
        gather_tiles([self.rgb, self.depth, self.trans], self.camera.width, self.camera.height,
                     self.group)
        vals, _ = self.loss(self.rgb, target, self.loss_cfg.mix, grad=self.dI,
                            want_value=want_loss)
        self._grad_pad.zero_()
        render_backward(s, self.camera, self.cfg, self.rgb, self.depth, self.trans, self.dI,
                        grad=self.grad, tile_begin=self.rank, tile_stride=self.world,
                        log=self.log)
        if self.rank == 0 and self.iso_cfg.lambda_s > 0:
            check(L.gsx_iso_loss(ptr(s.params), s.n, float(self.iso_cfg.r0),
                                 float(self.iso_cfg.lambda_s), ptr(self.grad), ptr(self._iso),
                                 stream_ptr()), "iso_loss")
        reduced = False
        if self.densify is not None:  # |dL/dmu| of this view (full gradient), before the update
            allreduce_grad(self._grad_pad, self.group)
            reduced = True
            self.densify.observe_view(self.grad, s.params, self.camera)
        self._optimizer_step(reduced)
        self._steps += 1
        if self.log is not None and (self._steps == 1 or want_loss):
            self.log.ensure()  # overflowed warps were replayed; size up for the next step
        if want_loss:
            s.check_render_status()  # a traversal-stack overflow since the last check
            iso = float(self._iso.item()) / s.n if self.rank == 0 else 0.0
            return vals[0] + self.iso_cfg.lambda_s * iso
        return None
