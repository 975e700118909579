"""Drop-in render entry points (renderer.py:263-500 of the reference) on the
B200 kernels.

`render` is the GPU-resident API (torch tensors in, torch tensors out, no host
synchronization).  `render_image` / `march_ray` / `march_rays` keep the
reference signatures and return host numpy arrays.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from ._lib import Stats, check, ptr, stream_ptr
from .config import Camera, Ray, RenderConfig, RenderStats


def _out(shape, out, device):
    if out is not None:
        return out
    return torch.empty(shape, dtype=torch.float32, device=device)


def render(scene, camera: Camera, cfg: RenderConfig | None = None, *, tile_begin: int = 0,
           tile_stride: int = 1, rgb=None, depth=None, trans=None, stats: bool = False,
           stream=None):
    """Render the 16x16 tiles tile_begin + k*tile_stride of `camera` into
    rgb [H,W,3], depth [H,W], trans [H,W] float32 CUDA tensors (allocated
    unless given).  Returns (rgb, depth, trans, stats_tensor_or_None)."""
    cfg = cfg or RenderConfig()
    L = _lib.lib()
    H, W = camera.height, camera.width
    dev = scene.device
    rgb = _out((H, W, 3), rgb, dev)
    depth = _out((H, W), depth, dev)
    trans = _out((H, W), trans, dev)
    st = torch.zeros(10, dtype=torch.int64, device=dev) if stats else None
    cam_c, cfg_c = camera.to_c(), cfg.to_c()
    import ctypes

    check(L.gsx_render_forward(ptr(scene.arena), ptr(scene.bvh_arena), scene.n,
                               ctypes.byref(cam_c), ctypes.byref(cfg_c), int(tile_begin),
                               int(tile_stride), ptr(rgb), ptr(depth), ptr(trans), ptr(st), None,
                               stream_ptr(stream)), "render_forward")
    return rgb, depth, trans, st


def render_backward(scene, camera: Camera, cfg: RenderConfig, rgb, depth, trans, dL_drgb,
                    dL_ddepth=None, dL_dtrans=None, *, grad=None, tile_begin: int = 0,
                    tile_stride: int = 1, stream=None):
    """Backward of `render` (no reference counterpart):
    accumulates dL/d(records) into grad [N,87] float32 (record layout, storage
    order; allocated zeroed unless given).  rgb/depth/trans are the forward
    outputs of the same tiles; dL_d* are the upstream gradients (CUDA tensors)."""
    import ctypes

    cfg = cfg or RenderConfig()
    L = _lib.lib()
    if grad is None:
        grad = torch.zeros((scene.n, 87), dtype=torch.float32, device=scene.device)
    cam_c, cfg_c = camera.to_c(), cfg.to_c()
    c = lambda t: None if t is None else t.contiguous()  # noqa: E731
    check(L.gsx_render_backward(ptr(scene.arena), ptr(scene.bvh_arena), ptr(scene.params), scene.n,
                                ctypes.byref(cam_c), ctypes.byref(cfg_c), int(tile_begin),
                                int(tile_stride), ptr(c(rgb)), ptr(c(depth)), ptr(c(trans)),
                                ptr(c(dL_drgb)), ptr(c(dL_ddepth)), ptr(c(dL_dtrans)), ptr(grad),
                                None, stream_ptr(stream)), "render_backward")
    return grad


def render_image(scene, camera: Camera, cfg: RenderConfig, threads: int | None = None):
    """renderer.py:396-437: returns (image (H,W,3) float64 numpy, RenderStats).
    `threads` / GSRAY_THREADS are accepted and ignored (one CUDA thread per ray)."""
    rgb, depth, trans, st = render(scene, camera, cfg, stats=True)
    stats = RenderStats.from_counts(st.cpu().numpy())
    return rgb.cpu().numpy().astype(np.float64), stats


def render_full(scene, camera: Camera, cfg: RenderConfig):
    """(rgb, depth, trans) as float64 numpy plus RenderStats."""
    rgb, depth, trans, st = render(scene, camera, cfg, stats=True)
    return (rgb.cpu().numpy().astype(np.float64), depth.cpu().numpy().astype(np.float64),
            trans.cpu().numpy().astype(np.float64), RenderStats.from_counts(st.cpu().numpy()))


def march_rays(scene, rays, cfg: RenderConfig, clip: bool = False, stats: bool = False):
    """Batch of explicit rays [M,8] (o, d, t_near, t_far) float64.  clip=False
    is march_ray semantics (renderer.py:263-285); clip=True applies
    clip_ray_to_scene first (render_image semantics).  Returns numpy
    rgb (M,3), depth (M,), trans (M,), RenderStats."""
    L = _lib.lib()
    dev = scene.device
    r = torch.as_tensor(np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 8), device=dev)
    m = r.shape[0]
    rgb = torch.empty((m, 3), dtype=torch.float32, device=dev)
    depth = torch.empty(m, dtype=torch.float32, device=dev)
    trans = torch.empty(m, dtype=torch.float32, device=dev)
    st = torch.zeros(10, dtype=torch.int64, device=dev) if stats else None
    import ctypes

    cfg_c = cfg.to_c()
    check(L.gsx_render_rays(ptr(scene.arena), ptr(scene.bvh_arena), scene.n, ptr(r), m,
                            int(bool(clip)), ctypes.byref(cfg_c), ptr(rgb), ptr(depth),
                            ptr(trans), ptr(st), None, stream_ptr()), "render_rays")
    s = RenderStats.from_counts(st.cpu().numpy()) if stats else None
    return (rgb.cpu().numpy().astype(np.float64), depth.cpu().numpy().astype(np.float64),
            trans.cpu().numpy().astype(np.float64), s)


def march_ray(scene, ray: Ray, cfg: RenderConfig, stats: RenderStats | None = None):
    """renderer.py:263-285: (rgb (3,), stats) with stats.transmittance set."""
    if stats is None:
        stats = RenderStats()
    rgb, depth, trans, s = march_rays(scene, ray.as_array()[None], cfg, clip=False, stats=True)
    stats.merge(s)
    stats.transmittance = float(trans[0])
    return rgb[0], stats


def clip_ray_to_scene(scene, ray: Ray) -> Ray | None:
    """renderer.py:160-175 (host mirror, float64)."""
    if ray.t_near >= ray.t_far:
        return None
    d = ray.direction
    inv = np.where(d == 0.0, np.inf, 1.0 / np.where(d == 0.0, 1.0, d))
    t0, t1 = -np.inf, np.inf
    for k in range(3):
        if d[k] != 0.0:
            a = (scene.bounds_lo[k] - ray.origin[k]) * inv[k]
            b = (scene.bounds_hi[k] - ray.origin[k]) * inv[k]
            if a > b:
                a, b = b, a
            t0, t1 = max(t0, a), min(t1, b)
        elif ray.origin[k] < scene.bounds_lo[k] or ray.origin[k] > scene.bounds_hi[k]:
            return None
    t0 = max(ray.t_near, t0)
    t1 = min(ray.t_far, t1)
    if t0 >= t1:
        return None
    return Ray(ray.origin, ray.direction, t0, t1)


def psnr(a, b, data_range: float = 1.0) -> float:
    """renderer.py:496-500."""
    mse = float(np.mean((np.asarray(a) - np.asarray(b)) ** 2))
    if mse == 0.0:
        return float("inf")
    return 10.0 * math.log10(data_range ** 2 / mse)
