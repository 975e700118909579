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
from .config import Camera, LazyRenderStats, Ray, RenderConfig, RenderStats


def _out(shape, out, device):
    if out is not None:
        return out
    return torch.empty(shape, dtype=torch.float32, device=device)


class MarchLog:
    """Device arena for the training forward's march log (include/gsx.h):
    the forward records each warp's candidate lists and per-sample sums, the
    backward consumes them instead of replaying the march.  Any capacity is
    correct (warps that do not fit are replayed); `usage()` reports what the
    last forward needed so `ensure()` can grow the arena."""

    def __init__(self, camera: Camera, *, tile_begin: int = 0, tile_stride: int = 1,
                 capacity: int | None = None, device="cuda"):
        import ctypes

        L = _lib.lib()
        self.tile_begin, self.tile_stride = int(tile_begin), int(tile_stride)
        cam_c = camera.to_c()
        self.min_bytes = int(L.gsx_march_log_min_bytes(ctypes.byref(cam_c), self.tile_begin,
                                                       self.tile_stride))
        if self.min_bytes < 0:
            raise ValueError("invalid camera / tile set for a march log")
        if capacity is None:  # C2 measured ~5 KiB per ray; 8 KiB leaves headroom
            rays = camera.width * camera.height // self.tile_stride
            capacity = self.min_bytes + 8192 * rays
        self.device = device
        self.arena = torch.empty(max(int(capacity), self.min_bytes), dtype=torch.uint8,
                                 device=device)

    @property
    def capacity(self) -> int:
        return self.arena.numel()

    def usage(self, stream=None):
        """(bytes the last logged forward needed, overflowed?) -- synchronizes."""
        import ctypes

        used, ovf = ctypes.c_int64(0), ctypes.c_int(0)
        check(_lib.lib().gsx_march_log_usage(ptr(self.arena), ctypes.byref(used),
                                             ctypes.byref(ovf), stream_ptr(stream)),
              "march_log_usage")
        return int(used.value), bool(ovf.value)

    def ensure(self, headroom: float = 1.25, stream=None) -> bool:
        """Grow the arena if the last forward overflowed it; True if grown."""
        used, ovf = self.usage(stream)
        if not ovf:
            return False
        self.arena = torch.empty(int(used * headroom), dtype=torch.uint8, device=self.device)
        return True


# Forward kernel variants (all give the same pixels; gsx_render_cfg.sums and
# the presence of a workspace select them): the silhouette-screened kernel
# with per-sample sums in shared memory (16 warps / SM, no spills) or in
# registers (32 warps / SM, spilled), and the unscreened packet-cone kernel.
# Which one is fastest depends on the device's memory latency -- measured
# across B200 boxes, the shared-memory kernel ranges from 8% faster to 14%
# slower than the unscreened one -- so `autotune` times them on the
# workload once and `render` uses the winner for that workload.
VARIANTS = {"screened": (True, 0), "screened-regs": (True, 1), "plain": (False, 0)}
_TUNED: dict = {}


def _tune_key(scene, camera: Camera, cfg: RenderConfig, logged: bool, tile_stride: int):
    return (scene.n, camera.width, camera.height, cfg.mode, bool(logged), int(tile_stride) > 1)


def autotune(scene, camera: Camera, cfg: RenderConfig | None = None, *, log=None,
             tile_begin: int = 0, tile_stride: int = 1, reps: int = 2) -> dict:
    """Time every forward variant on this workload (device events, after one
    warm-up each; synchronizes) and make the fastest the default of `render`
    for workloads of this shape.  Returns {variant: ms, "best": name}."""
    cfg = cfg or RenderConfig()
    H, W = camera.height, camera.width
    dev = scene.device
    bufs = (torch.empty((H, W, 3), device=dev), torch.empty((H, W), device=dev),
            torch.empty((H, W), device=dev))
    s = torch.cuda.current_stream()
    out = {}
    for name in VARIANTS:
        def run():
            render(scene, camera, cfg, tile_begin=tile_begin, tile_stride=tile_stride,
                   rgb=bufs[0], depth=bufs[1], trans=bufs[2], log=log, variant=name)
        run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            run()
        e1.record(s)
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / reps
    best = min(VARIANTS, key=lambda k: out[k])
    _TUNED[_tune_key(scene, camera, cfg, log is not None, tile_stride)] = best
    out["best"] = best
    return out


def render(scene, camera: Camera, cfg: RenderConfig | None = None, *, tile_begin: int = 0,
           tile_stride: int = 1, rgb=None, depth=None, trans=None, stats: bool = False,
           log: MarchLog | None = None, stream=None, screen: bool | None = None,
           traversal: int = 0, workspace=None, variant: str | None = None):
    """Render the 16x16 tiles tile_begin + k*tile_stride of `camera` into
    rgb [H,W,3], depth [H,W], trans [H,W] float32 CUDA tensors (allocated
    unless given).  Returns (rgb, depth, trans, stats_tensor_or_None).
    With `log` (training) the march is also recorded for render_backward.
    `variant` picks the forward kernel (VARIANTS; default: the one `autotune`
    chose for this workload shape, else "screened"); `screen=False` is
    variant "plain".  The screened kernels keep a per-camera silhouette table
    in `workspace` (default the scene's own render workspace -- pass separate
    ones for concurrent renders of one scene).  `traversal` forces the warp
    traversal (0 auto, 1 cone, 2 per-lane).  Pixels do not depend on any of
    these."""
    cfg = cfg or RenderConfig()
    L = _lib.lib()
    H, W = camera.height, camera.width
    dev = scene.device
    rgb = _out((H, W, 3), rgb, dev)
    depth = _out((H, W), depth, dev)
    trans = _out((H, W), trans, dev)
    st = torch.zeros(10, dtype=torch.int64, device=dev) if stats else None
    if variant is None:
        variant = "plain" if screen is False else _TUNED.get(
            _tune_key(scene, camera, cfg, log is not None, tile_stride), "screened")
    screen, sums = VARIANTS[variant]
    cam_c, cfg_c = camera.to_c(), cfg.to_c(traversal, sums)
    import ctypes

    if log is not None:
        if stats:
            raise ValueError("stats and log are exclusive")
        if (log.tile_begin, log.tile_stride) != (int(tile_begin), int(tile_stride)):
            raise ValueError("march log was sized for another tile set")
        ws = None
        if screen:
            ws = workspace if workspace is not None else scene.render_workspace()
        check(L.gsx_render_forward_logged(ptr(scene.arena), ptr(scene.bvh_arena), scene.n,
                                          ctypes.byref(cam_c), ctypes.byref(cfg_c),
                                          int(tile_begin), int(tile_stride), ptr(rgb),
                                          ptr(depth), ptr(trans), ptr(log.arena), log.capacity,
                                          ptr(ws), 0 if ws is None else ws.numel(),
                                          ptr(scene.render_status()), stream_ptr(stream)),
              "render_forward_logged")
        return rgb, depth, trans, None
    ws = None
    if screen and not stats:
        ws = workspace if workspace is not None else scene.render_workspace()
    check(L.gsx_render_forward(ptr(scene.arena), ptr(scene.bvh_arena), scene.n,
                               ctypes.byref(cam_c), ctypes.byref(cfg_c), int(tile_begin),
                               int(tile_stride), ptr(rgb), ptr(depth), ptr(trans), ptr(st),
                               ptr(ws), 0 if ws is None else ws.numel(),
                               ptr(scene.render_status()), stream_ptr(stream)), "render_forward")
    return rgb, depth, trans, st


def render_backward(scene, camera: Camera, cfg: RenderConfig, rgb, depth, trans, dL_drgb,
                    dL_ddepth=None, dL_dtrans=None, *, grad=None, tile_begin: int = 0,
                    tile_stride: int = 1, log: MarchLog | None = None, stream=None,
                    pass2: int = 0):
    """Backward of `render` (no reference counterpart):
    accumulates dL/d(records) into grad [N,87] float32 (record layout, storage
    order; allocated zeroed unless given).  rgb/depth/trans are the forward
    outputs of the same tiles; dL_d* are the upstream gradients (CUDA tensors).
    `log` = the MarchLog the forward of these outputs wrote (skips the replay);
    `pass2` forces its pass-2 strategy (0 auto from the log, 1 compacted
    (lane, primitive) pairs, 2 all lanes per entry; same gradients to fp32
    summation order)."""
    import ctypes

    cfg = cfg or RenderConfig()
    L = _lib.lib()
    if grad is None:
        grad = torch.zeros((scene.n, 87), dtype=torch.float32, device=scene.device)
    cam_c, cfg_c = camera.to_c(), cfg.to_c(pass2=pass2)
    c = lambda t: None if t is None else t.contiguous()  # noqa: E731
    if log is not None:
        if (log.tile_begin, log.tile_stride) != (int(tile_begin), int(tile_stride)):
            raise ValueError("march log was recorded for another tile set")
        check(L.gsx_render_backward_logged(
            ptr(scene.arena), ptr(scene.bvh_arena), ptr(scene.params), scene.n,
            ctypes.byref(cam_c), ctypes.byref(cfg_c), int(tile_begin), int(tile_stride),
            ptr(c(rgb)), ptr(c(depth)), ptr(c(trans)), ptr(c(dL_drgb)), ptr(c(dL_ddepth)),
            ptr(c(dL_dtrans)), ptr(log.arena), ptr(grad), ptr(scene.render_status()),
            stream_ptr(stream)), "render_backward_logged")
        return grad
    check(L.gsx_render_backward(ptr(scene.arena), ptr(scene.bvh_arena), ptr(scene.params), scene.n,
                                ctypes.byref(cam_c), ctypes.byref(cfg_c), int(tile_begin),
                                int(tile_stride), ptr(c(rgb)), ptr(c(depth)), ptr(c(trans)),
                                ptr(c(dL_drgb)), ptr(c(dL_ddepth)), ptr(c(dL_dtrans)), ptr(grad),
                                ptr(scene.render_status()), stream_ptr(stream)),
          "render_backward")
    return grad


def lazy_stats(scene, camera: Camera, cfg: RenderConfig) -> LazyRenderStats:
    """RenderStats of render_image(scene, camera, cfg), gathered by the STATS
    forward only when a counter is first read (see LazyRenderStats)."""
    version = scene.version

    def compute():
        if scene.version != version:
            raise RuntimeError("scene changed since the render; its RenderStats are gone")
        st = render(scene, camera, cfg, stats=True)[3]
        # (`transmittance` stays 1.0: render_image does not merge it,
        # renderer.py:79,85-93)
        return RenderStats.from_counts(st.cpu().numpy())

    return LazyRenderStats(compute)


def to_host64(t) -> np.ndarray:
    """float64 host copy of a float32 CUDA tensor: widened on the device, then
    one DMA into page-locked memory (torch's caching host allocator recycles
    the block once the returned array is gone)."""
    out = torch.empty(t.shape, dtype=torch.float64, pin_memory=True)
    out.copy_(t.double())
    return out.numpy()


def render_image(scene, camera: Camera, cfg: RenderConfig, threads: int | None = None):
    """renderer.py:396-437: returns (image (H,W,3) float64 numpy, RenderStats).
    `threads` / GSRAY_THREADS are accepted and ignored (one CUDA thread per ray).
    The image comes from the plain (screened) forward; the RenderStats are
    lazy: reading a counter runs the exact-counter pass then."""
    rgb, _, _, _ = render(scene, camera, cfg)
    img = to_host64(rgb)
    scene.check_render_status()
    return img, lazy_stats(scene, camera, cfg)


def render_full(scene, camera: Camera, cfg: RenderConfig):
    """(rgb, depth, trans) as float64 numpy plus (lazy) RenderStats."""
    rgb, depth, trans, _ = render(scene, camera, cfg)
    out = (to_host64(rgb), to_host64(depth), to_host64(trans))
    scene.check_render_status()
    return out + (lazy_stats(scene, camera, cfg),)


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
                            ptr(trans), ptr(st), ptr(scene.render_status()), stream_ptr()),
          "render_rays")
    s = RenderStats.from_counts(st.cpu().numpy()) if stats else None
    scene.check_render_status()
    return (rgb.cpu().numpy().astype(np.float64), depth.cpu().numpy().astype(np.float64),
            trans.cpu().numpy().astype(np.float64), s)


def ray_stats(scene, rays, cfg: RenderConfig, clip: bool = False):
    """Per-ray RenderStats counters of a batch of explicit rays [M,8]:
    int64 numpy [M,10] (rays, samples, segments, segments_skipped,
    closest_hit_calls, node_visits, aabb_hits, ellipsoid_hits, pairs,
    composited), march_ray semantics unless clip (gsx_render_rays_stats)."""
    import ctypes

    L = _lib.lib()
    dev = scene.device
    r = torch.as_tensor(np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 8), device=dev)
    m = r.shape[0]
    rgb = torch.empty((m, 3), dtype=torch.float32, device=dev)
    per = torch.zeros((m, 10), dtype=torch.int64, device=dev)
    cfg_c = cfg.to_c()
    check(L.gsx_render_rays_stats(ptr(scene.arena), ptr(scene.bvh_arena), scene.n, ptr(r), m,
                                  int(bool(clip)), ctypes.byref(cfg_c), ptr(rgb), None, None,
                                  ptr(per), ptr(scene.render_status()), stream_ptr()),
          "render_rays_stats")
    out = per.cpu().numpy()
    scene.check_render_status()
    return out


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


def reference_rays(scene, rays, fine_dt: float, background=(0.0, 0.0, 0.0),
                   clip: bool = False) -> np.ndarray:
    """Dense all-primitive quadrature of a batch of rays [M,8] (o, d, t_near,
    t_far) on the device, float64 (gsx_reference_rays): reference_integrate
    per ray, after clip_ray_to_scene when `clip` (reference_render)."""
    import ctypes

    L = _lib.lib()
    dev = scene.device
    r = torch.as_tensor(np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 8), device=dev)
    bg = (ctypes.c_double * 3)(*[float(v) for v in background])
    out = torch.empty((r.shape[0], 3), dtype=torch.float64, device=dev)
    check(L.gsx_reference_rays(ptr(scene.arena), ptr(scene.params), scene.n, ptr(r), r.shape[0],
                               int(bool(clip)), float(fine_dt), bg, ptr(out), stream_ptr()),
          "reference_rays")
    return out.cpu().numpy()


def reference_integrate(scene, ray: Ray, fine_dt: float, background=(0.0, 0.0, 0.0)):
    """renderer.py:440-480: dense uniform quadrature of one ray over its
    [t_near, t_far] against every primitive (no BVH, no skipping) -- the
    oracle the renderer's tests compare against.  Returns rgb (3,) float64."""
    return reference_rays(scene, ray.as_array()[None], fine_dt, background, clip=False)[0]


def reference_render(scene, camera: Camera, fine_dt: float, background=(0.0, 0.0, 0.0)):
    """renderer.py:483-493: reference_integrate per pixel with render_image's
    ray clipping; (H,W,3) float64."""
    img = reference_rays(scene, camera.rays(), fine_dt, background, clip=True)
    return img.reshape(camera.height, camera.width, 3)


def psnr(a, b, data_range: float = 1.0) -> float:
    """renderer.py:496-500."""
    mse = float(np.mean((np.asarray(a) - np.asarray(b)) ** 2))
    if mse == 0.0:
        return float("inf")
    return 10.0 * math.log10(data_range ** 2 / mse)
