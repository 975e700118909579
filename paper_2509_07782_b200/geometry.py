"""Primitive value types and closed-form ellipsoid geometry (the public names
of the reference's geometry.py:67-233), as host float64 helpers around the
[N,87] record layout the device path consumes.

Every function works on one shape (the reference's signature) and, through
the `*_batch` forms, on arrays of scales / rotations at once.  The training
regularizer `isotropic_loss` runs on the device (K9, gsx_iso_loss) for a list
of shapes or a [N,87] record tensor alike.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .config import quat_to_rotation
from .errors import EmptyIsosurface, EmptyScene
from .loss import SPHERE_RATIO, IsoLossConfig

S_MIN = 1e-7  # geometry.py:21: scales are clamped here before any geometry op


@dataclass(frozen=True)
class GaussianShape:
    """geometry.py:67-87: mean, scalar-first unit quaternion (normalized on
    ingestion), per-axis scales clamped at S_MIN, amplitude sigma~ >= 0."""

    mean: np.ndarray
    quat: np.ndarray
    scales: np.ndarray
    sigma: float
    rotation: np.ndarray = field(init=False, repr=False)

    def __post_init__(self):
        if self.sigma < 0:
            raise ValueError("sigma must be nonnegative")
        q = np.asarray(self.quat, dtype=float).reshape(4)
        q = q / np.linalg.norm(q)
        object.__setattr__(self, "mean", np.asarray(self.mean, dtype=float).reshape(3))
        object.__setattr__(self, "quat", q)
        object.__setattr__(self, "scales",
                           np.maximum(np.asarray(self.scales, dtype=float).reshape(3), S_MIN))
        object.__setattr__(self, "rotation", quat_to_rotation(q))

    def record_head(self) -> np.ndarray:
        """The geometric 11 floats of the 87-float record (scene_io.py:26-44)."""
        return np.concatenate([self.mean, self.quat, self.scales, [float(self.sigma)]])


@dataclass(frozen=True)
class Aabb:
    """geometry.py:90-104."""

    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.lo, dtype=float).reshape(3)
        hi = np.asarray(self.hi, dtype=float).reshape(3)
        if np.any(lo > hi):
            raise ValueError("AABB min corner exceeds max corner")
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)

    def volume(self) -> float:
        return float(np.prod(self.hi - self.lo))


def _log_ratio(shape: GaussianShape, sigma_eps: float) -> float:
    if sigma_eps <= 0:
        raise ValueError("sigma_eps must be positive")
    if shape.sigma <= sigma_eps:
        raise EmptyIsosurface(
            f"amplitude {shape.sigma} <= threshold {sigma_eps}: empty isosurface")
    return 2.0 * math.log(shape.sigma / sigma_eps)


def iso_scale(shape: GaussianShape, sigma_eps: float) -> np.ndarray:
    """geometry.py:124-137: semi-axes of the sigma = sigma_eps level set,
    sqrt(2 ln(sigma~ / sigma_eps)) * scales."""
    return math.sqrt(_log_ratio(shape, sigma_eps)) * shape.scales


def aabb_of(shape: GaussianShape, sigma_eps: float) -> Aabb:
    """geometry.py:140-149: minimal box of the bounding ellipsoid; the half
    extent along world axis i is |row_i(R) * s~| (the kernels' K1 formula)."""
    half = np.sqrt(((shape.rotation * iso_scale(shape, sigma_eps)) ** 2).sum(axis=1))
    return Aabb(shape.mean - half, shape.mean + half)


def ellipsoid_volume(shape: GaussianShape, sigma_eps: float) -> float:
    """geometry.py:168-177: (4 pi / 3) k^(3/2) s1 s2 s3."""
    k = _log_ratio(shape, sigma_eps)
    return (4.0 * math.pi / 3.0) * k ** 1.5 * float(np.prod(shape.scales))


def volume_ratio_batch(rotations, scales) -> np.ndarray:
    """AABB / ellipsoid volume for (N,3,3) rotations and (N,3) scales:
    (6/pi) sqrt(prod_i sum_j R_ij^2 s_j^2) / prod_j s_j (independent of the
    level-set factor, geometry.py:180-190)."""
    s = np.maximum(np.asarray(scales, dtype=float).reshape(-1, 3), S_MIN)
    r2 = np.asarray(rotations, dtype=float).reshape(-1, 3, 3) ** 2
    return SPHERE_RATIO * np.sqrt(np.prod(r2 @ (s ** 2)[..., None], axis=(1, 2))) / s.prod(axis=1)


def volume_ratio(shape: GaussianShape, sigma_eps: float | None = None) -> float:
    """geometry.py:180-190 (sigma_eps accepted for symmetry and ignored)."""
    return float(volume_ratio_batch(shape.rotation[None], shape.scales[None])[0])


def ratio_upper_bound_batch(scales) -> np.ndarray:
    """Rotation-independent bound (2 / (pi sqrt 3)) |s|^3 / (s1 s2 s3) for
    (N,3) scales (geometry.py:193-202)."""
    s = np.maximum(np.asarray(scales, dtype=float).reshape(-1, 3), S_MIN)
    return (2.0 / (math.pi * math.sqrt(3.0))) * (s ** 2).sum(axis=1) ** 1.5 / s.prod(axis=1)


def ratio_upper_bound(scales) -> float:
    """geometry.py:193-202."""
    return float(ratio_upper_bound_batch(scales)[0])


def ratio_upper_bound_gradient(scales) -> np.ndarray:
    """geometry.py:205-212: d r_max / d s_k = r_max (3 s_k / |s|^2 - 1 / s_k)."""
    s = np.maximum(np.asarray(scales, dtype=float).reshape(3), S_MIN)
    return ratio_upper_bound(s) * (3.0 * s / (s ** 2).sum() - 1.0 / s)


def isotropic_loss(shapes, cfg: IsoLossConfig = IsoLossConfig()):
    """geometry.py:215-233: (L_s, dL_s/ds (N,3)) -- the mean hinge
    max(r_max - r0, 0) over the shapes and its gradient (zero at r_max = r0).

    `shapes` is a list of GaussianShape (the reference's form: their scales
    are packed into records and evaluated by the device kernel) or an [N,87]
    CUDA record tensor (the training form, see loss.isotropic_loss)."""
    import torch

    from . import loss as _loss

    if isinstance(shapes, torch.Tensor):
        val, g = _loss.isotropic_loss(shapes, cfg)
        return val, g[:, 7:10]
    if len(shapes) == 0:
        raise EmptyScene("isotropic loss of an empty primitive list")
    rec = torch.zeros((len(shapes), 87), dtype=torch.float32, device="cuda")
    rec[:, 7:10] = torch.as_tensor(np.stack([s.scales for s in shapes]), dtype=torch.float32)
    val, g = _loss.isotropic_loss(rec, cfg)
    return val, g[:, 7:10].double().cpu().numpy()
