"""Densification statistics on the device (densify.py of the reference).

`GradAccumulator`, `criterion_old`, `criterion_new`, `DensifyConfig` and
`observe_scene` keep the reference names and semantics (densify.py:28-83,
190-204).  The difference is where the per-primitive gradient comes from:
the reference finite-differences the image loss w.r.t. every mean (6 renders
per primitive per camera, fd_position_gradient densify.py:156-187); here one
render + loss + backward yields dL/dmu for all primitives at once, and
`gsx_densify_observe` (csrc/densify.cu) accumulates |dL/dmu| and
alpha |dL/dmu| (alpha = |mu - camera center| / focal) in float64.

The accumulator is plain bookkeeping over three device tensors; the scalar
`observe` / `merge` calls mirror the reference API and work on any device,
the per-view observation and the criteria run as CUDA kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check, ptr, stream_ptr
from .loss import LossConfig


@dataclass(frozen=True)
class DensifyConfig:
    """densify.py:28-36."""

    tau: float = 0.00015
    window: int = 100
    radius: float = 0.125

    def __post_init__(self):
        if self.tau <= 0 or self.radius <= 0 or self.window < 1:
            raise ValueError("tau and radius must be positive, window >= 1")


class GradAccumulator:
    """Per-primitive sums of raw and alpha-weighted gradient norms
    (densify.py:49-66): sum_raw, sum_weighted float64 [N], counts int64 [N]."""

    def __init__(self, n_primitives: int, device="cuda"):
        self.sum_raw = torch.zeros(n_primitives, dtype=torch.float64, device=device)
        self.sum_weighted = torch.zeros(n_primitives, dtype=torch.float64, device=device)
        self.counts = torch.zeros(n_primitives, dtype=torch.int64, device=device)

    def __len__(self):
        return self.counts.numel()

    def observe(self, index: int, grad_norm: float, alpha: float):
        """One scalar observation (densify.py:55-61)."""
        if grad_norm < 0 or alpha < 0:
            raise ValueError("norms and weights must be nonnegative")
        self.sum_raw[index] += grad_norm
        self.sum_weighted[index] += alpha * grad_norm
        self.counts[index] += 1

    def merge(self, other: "GradAccumulator"):
        """densify.py:63-66 (also the cross-rank merge of per-rank views)."""
        self.sum_raw += other.sum_raw
        self.sum_weighted += other.sum_weighted
        self.counts += other.counts

    def reset(self):
        self.sum_raw.zero_()
        self.sum_weighted.zero_()
        self.counts.zero_()

    def observe_view(self, grad, params, camera, indices=None, stream=None):
        """Observe one camera from the backward's gradient grad [N,87] (record
        layout; after the multi-GPU all-reduce): |dL/dmu_i| and
        alpha_i = |mu_i - center| / focal for every primitive (or `indices`)."""
        L = _lib.lib()
        n = len(self)
        if grad.shape != (n, 87) or params.shape != (n, 87):
            raise ValueError("grad and params must be [N,87] for this accumulator")
        idx = None
        m = n
        if indices is not None:
            idx = torch.as_tensor(indices, dtype=torch.int64, device=self.counts.device)
            m = idx.numel()
        center = (ctypes.c_double * 3)(*[float(x) for x in camera.center])
        check(L.gsx_densify_observe(ptr(grad.contiguous()), ptr(params.contiguous()), n, ptr(idx),
                                    m, center, float(camera.focal), ptr(self.sum_raw),
                                    ptr(self.sum_weighted), ptr(self.counts), stream_ptr(stream)),
              "densify_observe")


def _criterion(acc: GradAccumulator, cfg: DensifyConfig, weighted: bool):
    n = len(acc)
    out = torch.zeros(n, dtype=torch.uint8, device=acc.counts.device)
    if acc.counts.device.type == "cuda":
        L = _lib.lib()
        check(L.gsx_densify_criteria(ptr(acc.sum_raw), ptr(acc.sum_weighted), ptr(acc.counts), n,
                                     float(cfg.tau), None if weighted else ptr(out),
                                     ptr(out) if weighted else None, stream_ptr()),
              "densify_criteria")
        return out.bool()
    # host bookkeeping (CPU tensors): the same strict comparison
    seen = acc.counts >= 1
    s = acc.sum_weighted if weighted else acc.sum_raw
    mean = torch.where(seen, s / acc.counts.clamp(min=1).double(), torch.zeros_like(s))
    return seen & (mean > cfg.tau)


def criterion_old(acc: GradAccumulator, cfg: DensifyConfig):
    """Mean unweighted gradient norm exceeds tau; False with no observations
    (densify.py:69-74).  Returns a bool tensor [N]."""
    return _criterion(acc, cfg, weighted=False)


def criterion_new(acc: GradAccumulator, cfg: DensifyConfig):
    """Mean alpha-weighted gradient norm exceeds tau (densify.py:77-82)."""
    return _criterion(acc, cfg, weighted=True)


def _point_records(pts):
    """Degenerate primitives at the given points (s = S_MIN, unit sigma~): the
    BVH over their boxes is a BVH over the points."""
    import numpy as np

    rec = np.zeros((len(pts), 87), dtype=np.float32)
    rec[:, 0:3] = pts
    rec[:, 3] = 1.0
    rec[:, 7:10] = 1e-7
    rec[:, 10] = 1.0
    rec[:, 40::3][:, :7] = 1.0  # SG axes (0, 0, 1): valid, never evaluated
    return rec


def neighbor_density(means, radius: float):
    """Number of other points within the closed ball of the given radius
    (densify.py:86-97, cKDTree.query_ball_point minus self), on the GPU over
    the scene BVH (`gsx_neighbor_density`).  `means` is a Scene (uses its
    means and BVH; returns an int64 device tensor in storage order) or an
    [N,3] array (rounded to float32 like a .gsx record; returns numpy)."""
    import numpy as np

    from .scene import Scene

    if radius <= 0:
        raise ValueError("radius must be positive")
    as_numpy = not isinstance(means, Scene)
    scene = means if not as_numpy else Scene.from_records(
        _point_records(np.asarray(means, dtype=float).reshape(-1, 3)))
    L = _lib.lib()
    counts = torch.empty(scene.n, dtype=torch.int64, device=scene.device)
    st = _lib.new_status(scene.device)
    check(L.gsx_neighbor_density(ptr(scene.arena), ptr(scene.bvh_arena), scene.n, float(radius),
                                 ptr(counts), ptr(st), stream_ptr()), "neighbor_density")
    _lib.raise_status(st, "neighbor_density")
    return counts.cpu().numpy() if as_numpy else counts


def fd_position_gradient(scene, camera, target, index: int, h: float | None = None,
                         loss_cfg: LossConfig | None = None, render_cfg=None,
                         iso_loss: float = 0.0):
    """densify.py:156-187: central-difference gradient of the image loss
    w.r.t. primitive `index`'s mean (storage index), by six device renders of
    `scene.with_mean` copies (each a full K1-K5 rebuild, as the reference
    rebuilds its Scene and BVH).  Renders default to uniform mode, the step
    to 1e-4 x the scene diagonal.  The analytic gradient of the same loss is
    `render_backward` (observe_scene uses it); this is the reference's
    finite-difference API, e.g. to cross-check it."""
    import numpy as np

    from .config import RenderConfig
    from .loss import image_loss
    from .renderer import render

    loss_cfg = loss_cfg or LossConfig()
    render_cfg = render_cfg or RenderConfig(mode="uniform")
    if h is None:
        h = 1e-4 * float(np.linalg.norm(scene.bounds_hi - scene.bounds_lo))
    mu = scene.params[index, 0:3].double().cpu().numpy()
    tgt = torch.as_tensor(np.asarray(target, dtype=np.float32), device=scene.device)
    grad = np.zeros(3)
    for axis in range(3):
        step = np.zeros(3)
        step[axis] = h
        losses, xs = [], []
        for sgn in (1.0, -1.0):
            m = (mu + sgn * step).astype(np.float32)  # the records are float32
            img = render(scene.with_mean(index, m), camera, render_cfg)[0]
            losses.append(image_loss(img, tgt, loss_cfg, iso_loss))
            xs.append(float(m[axis]))
        grad[axis] = (losses[0] - losses[1]) / (xs[0] - xs[1])
    return grad


def observe_scene(acc: GradAccumulator, scene, camera, target, indices=None,
                  loss_cfg: LossConfig | None = None, render_cfg=None):
    """Record one camera observation (densify.py:190-204): render, image loss,
    analytic backward, then |dL/dmu| and alpha for every primitive (or
    `indices`).  Like the reference, renders default to uniform mode."""
    from .config import RenderConfig
    from .loss import image_loss_grad
    from .renderer import render, render_backward

    loss_cfg = loss_cfg or LossConfig()
    render_cfg = render_cfg or RenderConfig(mode="uniform")
    dev = scene.device
    tgt = torch.as_tensor(target, dtype=torch.float32, device=dev)
    rgb, depth, trans, _ = render(scene, camera, render_cfg)
    _, dI = image_loss_grad(rgb, tgt, loss_cfg.mix)
    grad = render_backward(scene, camera, render_cfg, rgb, depth, trans, dI)
    acc.observe_view(grad, scene.params, camera, indices)
    return grad
