"""Training losses on the device: image loss (L1 + DSSIM, densify.py:99-153)
and the isotropic regularizer (geometry.py:107-233), with their gradients.

Kernels: gsx_image_loss (K8) and gsx_iso_loss (K9) in csrc/loss.cu."""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr, stream_ptr

SPHERE_RATIO = 6.0 / np.pi


@dataclass(frozen=True)
class LossConfig:
    """densify.py:39-46."""

    mix: float = 0.2
    lambda_s: float = 0.00025

    def __post_init__(self):
        if not (0.0 <= self.mix <= 1.0):
            raise ValueError("mix must be in [0, 1]")


@dataclass(frozen=True)
class IsoLossConfig:
    """geometry.py:107-121."""

    lambda_s: float = 0.00025
    r0: float = 10.0

    def __post_init__(self):
        if self.lambda_s < 0:
            raise ValueError("lambda_s must be nonnegative")
        if self.r0 < SPHERE_RATIO:
            raise ValueError(f"r0 must be >= 6/pi ({SPHERE_RATIO:.6f})")


class ImageLoss:
    """Reusable workspace for the fused image loss of [H, W, C] images."""

    def __init__(self, h: int, w: int, c: int = 3, device=None):
        self.shape = (h, w, c)
        L = _lib.lib()
        self.ws = torch.empty(L.gsx_image_loss_workspace_bytes(h, w, c), dtype=torch.uint8,
                              device=device or "cuda")

    def __call__(self, rendered, target, mix: float = 0.2, grad=None, want_value: bool = True):
        """Returns ((loss, l1, ssim) or None, dL/drendered tensor or None)."""
        L = _lib.lib()
        h, w, c = self.shape
        out = (ctypes.c_double * 3)()
        check(L.gsx_image_loss(ptr(rendered.contiguous()), ptr(target.contiguous()), h, w, c,
                               float(mix), ptr(grad), out if want_value else None, ptr(self.ws),
                               stream_ptr()), "image_loss")
        vals = (out[0], out[1], out[2]) if want_value else None
        return vals, grad


def _as_image(a, device):
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a, dtype=np.float32))
    t = t.to(device=device, dtype=torch.float32)
    if t.ndim == 2:
        t = t[..., None]
    return t.contiguous()


def image_loss(rendered, target, cfg: LossConfig = LossConfig(), iso_loss: float = 0.0) -> float:
    """densify.py:139-153: (1-mix) L1 + mix DSSIM + lambda_s iso_loss (GPU)."""
    r = _as_image(rendered, "cuda")
    t = _as_image(target, "cuda")
    if r.shape != t.shape:
        raise ValueError("image shapes differ")
    vals, _ = ImageLoss(*r.shape)(r, t, cfg.mix)
    return vals[0] + cfg.lambda_s * iso_loss


def ssim(a, b) -> float:
    r = _as_image(a, "cuda")
    t = _as_image(b, "cuda")
    if r.shape != t.shape:
        raise ValueError("image shapes differ")
    return ImageLoss(*r.shape)(r, t, 1.0)[0][2]


def dssim(a, b) -> float:
    """densify.py:135-136."""
    return (1.0 - ssim(a, b)) / 2.0


def image_loss_grad(rendered, target, mix: float = 0.2):
    """(loss value, dL/d rendered) for [H,W,C] CUDA tensors."""
    r = _as_image(rendered, "cuda")
    t = _as_image(target, "cuda")
    g = torch.empty_like(r)
    vals, g = ImageLoss(*r.shape)(r, t, mix, grad=g)
    return vals[0], g


def isotropic_loss(params, cfg: IsoLossConfig = IsoLossConfig(), grad=None):
    """geometry.py:215-233 over [N,87] records (CUDA).  Returns (L_s, grad):
    grad [N,87] receives lambda_s dL_s/ds in the scale slots (accumulated if
    given, else a new tensor holding dL_s/ds, i.e. lambda_s = 1)."""
    L = _lib.lib()
    n = params.shape[0]
    own = grad is None
    if own:
        grad = torch.zeros_like(params)
    lam = 1.0 if own else cfg.lambda_s
    acc = torch.zeros(1, dtype=torch.float64, device=params.device)
    check(L.gsx_iso_loss(ptr(params), n, float(cfg.r0), float(lam), ptr(grad), ptr(acc),
                         stream_ptr()), "iso_loss")
    return float(acc.item()) / n, grad
