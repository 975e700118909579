"""View-dependent radiance and the mixture fields (the public names of the
reference's appearance.py:19-134).

`AppearanceCoeffs` / `eval_radiance` are host float64 value helpers for one
primitive (the device evaluates the same formula inside the march,
render_common.cuh eval_radiance_pre); `eval_fields` queries the mixture on
the device (gsx_eval_fields, float64, csrc/dense.cu) -- one point per call
like the reference, or many at once through `eval_fields_batch`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr, stream_ptr

N_SH, N_SG = 9, 7
_Y0 = 0.5 * math.sqrt(1.0 / math.pi)
_Y1 = math.sqrt(3.0 / (4.0 * math.pi))
_Y2XY = 0.5 * math.sqrt(15.0 / math.pi)
_Y2Z = 0.25 * math.sqrt(5.0 / math.pi)
_Y2XX = 0.25 * math.sqrt(15.0 / math.pi)


def sh_basis(d) -> np.ndarray:
    """Real SH basis to degree 2 at unit direction(s) d (3,) or (N,3), band
    order Y00; Y1-1, Y10, Y11; Y2-2 .. Y22 (appearance.py:26-50)."""
    d = np.asarray(d, dtype=float)
    x, y, z = d[..., 0], d[..., 1], d[..., 2]
    return np.stack([np.full_like(x, _Y0), _Y1 * y, _Y1 * z, _Y1 * x, _Y2XY * x * y,
                     _Y2XY * y * z, _Y2Z * (3.0 * z * z - 1.0), _Y2XY * x * z,
                     _Y2XX * (x * x - y * y)], axis=-1)


@dataclass(frozen=True)
class AppearanceCoeffs:
    """appearance.py:53-88: 9x3 SH coefficients and 7 spherical-Gaussian lobes
    (unit axis, sharpness >= 0, RGB amplitude); axes normalized on ingestion."""

    sh: np.ndarray
    sg_axis: np.ndarray
    sg_sharp: np.ndarray
    sg_amp: np.ndarray

    def __post_init__(self):
        axis = np.asarray(self.sg_axis, dtype=float).reshape(N_SG, 3)
        norm = np.linalg.norm(axis, axis=1)
        if np.any(norm < 1e-12):
            raise ValueError("SG lobe axis must be nonzero")
        sharp = np.asarray(self.sg_sharp, dtype=float).reshape(N_SG)
        if np.any(sharp < 0):
            raise ValueError("SG sharpness must be nonnegative")
        object.__setattr__(self, "sh", np.asarray(self.sh, dtype=float).reshape(N_SH, 3))
        object.__setattr__(self, "sg_axis", axis / norm[:, None])
        object.__setattr__(self, "sg_sharp", sharp)
        object.__setattr__(self, "sg_amp", np.asarray(self.sg_amp, dtype=float).reshape(N_SG, 3))

    @classmethod
    def constant(cls, rgb) -> "AppearanceCoeffs":
        """Direction-independent radiance: the DC coefficient only."""
        sh = np.zeros((N_SH, 3))
        sh[0] = np.asarray(rgb, dtype=float) / _Y0
        return cls(sh=sh, sg_axis=np.tile([0.0, 0.0, 1.0], (N_SG, 1)),
                   sg_sharp=np.zeros(N_SG), sg_amp=np.zeros((N_SG, 3)))

    def record_tail(self) -> np.ndarray:
        """The 76 appearance floats of the 87-float record (scene_io.py:26-44)."""
        return np.concatenate([self.sh.ravel(), self.sg_axis.ravel(), self.sg_sharp,
                               self.sg_amp.ravel()])


def eval_radiance(coeffs: AppearanceCoeffs, d) -> np.ndarray:
    """appearance.py:91-98: SH + sum_k a_k exp(lambda_k (nu_k . d - 1)),
    clamped at zero after the sum."""
    d = np.asarray(d, dtype=float).reshape(3)
    lobes = np.exp(coeffs.sg_sharp * (coeffs.sg_axis @ d - 1.0))
    return np.maximum(sh_basis(d) @ coeffs.sh + lobes @ coeffs.sg_amp, 0.0)


@dataclass(frozen=True)
class FieldSample:
    """appearance.py:101-104."""

    sigma: float
    color: np.ndarray


def eval_fields_batch(scene, points, dirs, active=None):
    """Mixture density (M,) and density-weighted radiance (M,3), float64, at
    points [M,3] for directions [M,3] over every primitive or the storage
    indices `active` (gsx_eval_fields)."""
    L = _lib.lib()
    dev = scene.device
    x = torch.as_tensor(np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3), device=dev)
    d = torch.as_tensor(np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3), device=dev)
    if x.shape != d.shape:
        raise ValueError("points and directions differ in count")
    a = None
    if active is not None:
        a = torch.as_tensor(np.asarray(active, dtype=np.int64).reshape(-1), device=dev)
    m = x.shape[0]
    sigma = torch.empty(m, dtype=torch.float64, device=dev)
    color = torch.empty((m, 3), dtype=torch.float64, device=dev)
    st = _lib.new_status(dev)
    check(L.gsx_eval_fields(ptr(scene.arena), ptr(scene.params), scene.n, ptr(x), ptr(d), m,
                            ptr(a), 0 if a is None else a.numel(), ptr(sigma), ptr(color),
                            ptr(st), stream_ptr()), "eval_fields")
    _lib.raise_status(st, "eval_fields")
    return sigma.cpu().numpy(), color.cpu().numpy()


def eval_fields(scene, x, d, active=None) -> FieldSample:
    """appearance.py:107-134: density and radiance of the mixture at point x
    for direction d; `active` narrows it to those storage indices (primitives
    whose bounding ellipsoid does not contain x contribute nothing, so any
    superset gives the same result).  Zero density is black."""
    sigma, color = eval_fields_batch(scene, np.asarray(x, float)[None], np.asarray(d, float)[None],
                                     active)
    return FieldSample(float(sigma[0]), color[0])
