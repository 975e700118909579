"""Configuration and value types mirroring the reference renderer's
(renderer.py:27-145): same field names, defaults and validation errors."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from ._lib import CameraC, RenderCfg


@dataclass(frozen=True)
class RenderConfig:
    """renderer.py:27-49.  `tile_size` and `buffer_capacity` are accepted for
    signature compatibility: pixels are tile-size invariant and overflow
    splitting is bitwise neutral in the reference (renderer.py:361-371), so the
    GPU path processes candidates in unbounded streams instead."""

    dt: float = 0.0025
    n_s: int = 16
    t_eps: float = 1e-4
    mode: str = "uniform"
    beta: float = 1024.0
    dt_min: float = 0.005
    dt_max: float = 0.02
    ess: bool = True
    tile_size: int = 16
    background: tuple = (0.0, 0.0, 0.0)
    buffer_capacity: int = 64

    def __post_init__(self):
        if not (0.0 < self.t_eps < 1.0):
            raise ValueError("t_eps must be in (0, 1)")
        if self.n_s < 1:
            raise ValueError("n_s must be >= 1")
        if self.dt_min > self.dt_max:
            raise ValueError("dt_min must be <= dt_max")
        if self.mode not in ("uniform", "adaptive"):
            raise ValueError(f"unknown mode {self.mode!r}")

    def to_c(self, traversal: int = 0, sums: int = 0, pass2: int = 0) -> RenderCfg:
        """C mirror (include/gsx.h gsx_render_cfg); `traversal`, `sums` and
        `pass2` are the extension fields (traversal: 0 by focal length, 1
        packet cone, 2 per-lane; sums of the screened forward: 0 shared memory,
        1 registers; pass 2 of the logged backward: 0 auto, 1 pairs, 2 all
        lanes per entry)."""
        c = RenderCfg()
        c.traversal = int(traversal)
        c.sums = int(sums)
        c.pass2 = int(pass2)
        c.dt, c.n_s, c.t_eps = float(self.dt), int(self.n_s), float(self.t_eps)
        c.mode = 1 if self.mode == "adaptive" else 0
        c.beta, c.dt_min, c.dt_max = float(self.beta), float(self.dt_min), float(self.dt_max)
        c.ess, c.tile_size = int(bool(self.ess)), int(self.tile_size)
        for k in range(3):
            c.background[k] = float(self.background[k])
        c.buffer_capacity = int(self.buffer_capacity)
        return c


@dataclass(frozen=True)
class Ray:
    """renderer.py:52-66."""

    origin: np.ndarray
    direction: np.ndarray
    t_near: float
    t_far: float

    def __post_init__(self):
        o = np.asarray(self.origin, dtype=float).reshape(3)
        d = np.asarray(self.direction, dtype=float).reshape(3)
        n = np.linalg.norm(d)
        if abs(n - 1.0) > 1e-9:
            d = d / n
        object.__setattr__(self, "origin", o)
        object.__setattr__(self, "direction", d)

    def as_array(self) -> np.ndarray:
        return np.concatenate([self.origin, self.direction, [self.t_near, self.t_far]])


def quat_to_rotation(q) -> np.ndarray:
    """geometry.py:26-42."""
    q = np.asarray(q, dtype=float)
    n = np.linalg.norm(q)
    if n < 1e-12:
        raise ValueError("zero quaternion")
    w, x, y, z = q / n
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


@dataclass(frozen=True)
class Camera:
    """Pinhole camera (renderer.py:109-145): scalar-first camera-to-world quat,
    looks along local +z, +y down; rays through pixel centres."""

    center: np.ndarray
    quat: np.ndarray
    focal: float
    width: int
    height: int
    t_near: float = 1e-4
    t_far: float = 1e6

    def __post_init__(self):
        if self.focal <= 0:
            raise ValueError("focal must be positive")
        if self.width < 1 or self.height < 1:
            raise ValueError("image dimensions must be >= 1")
        object.__setattr__(self, "center", np.asarray(self.center, dtype=float).reshape(3))
        q = np.asarray(self.quat, dtype=float).reshape(4)
        object.__setattr__(self, "quat", q / np.linalg.norm(q))
        object.__setattr__(self, "rotation", quat_to_rotation(self.quat))

    def ray(self, px: int, py: int) -> Ray:
        d_cam = np.array([(px + 0.5 - 0.5 * self.width) / self.focal,
                          (py + 0.5 - 0.5 * self.height) / self.focal, 1.0])
        d = self.rotation @ d_cam
        d = d / np.linalg.norm(d)
        return Ray(self.center, d, self.t_near, self.t_far)

    def rays(self, pixels=None) -> np.ndarray:
        """[M,8] float64 (o, d, t_near, t_far) of the given (px, py) pixels
        (all pixels, row-major, when None) -- Camera.ray vectorised."""
        if pixels is None:
            py, px = np.mgrid[0:self.height, 0:self.width]
            pixels = np.stack([px.ravel(), py.ravel()], axis=1)
        pix = np.asarray(pixels, dtype=np.float64).reshape(-1, 2)
        d_cam = np.stack([(pix[:, 0] + 0.5 - 0.5 * self.width) / self.focal,
                          (pix[:, 1] + 0.5 - 0.5 * self.height) / self.focal,
                          np.ones(len(pix))], axis=1)
        d = d_cam @ self.rotation.T
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        out = np.empty((len(pix), 8))
        out[:, 0:3] = self.center
        out[:, 3:6] = d
        out[:, 6] = self.t_near
        out[:, 7] = self.t_far
        return out

    def to_c(self) -> CameraC:
        c = CameraC()
        R = np.ascontiguousarray(self.rotation, dtype=np.float64).ravel()
        for k in range(9):
            c.R[k] = float(R[k])
        for k in range(3):
            c.center[k] = float(self.center[k])
        c.focal = float(self.focal)
        c.width, c.height = int(self.width), int(self.height)
        c.t_near, c.t_far = float(self.t_near), float(self.t_far)
        return c

    @property
    def n_tiles(self) -> int:
        return ((self.width + 15) // 16) * ((self.height + 15) // 16)


_STAT_KEYS = ("rays", "samples", "segments", "segments_skipped", "closest_hit_calls",
              "node_visits", "aabb_hits", "ellipsoid_hits")


@dataclass
class RenderStats:
    """renderer.py:69-106.  `node_visits` counts visits of the LBVH, which has a
    different topology from the reference's SAH tree."""

    rays: int = 0
    samples: int = 0
    segments: int = 0
    segments_skipped: int = 0
    closest_hit_calls: int = 0
    node_visits: int = 0
    aabb_hits: int = 0
    ellipsoid_hits: int = 0
    transmittance: float = 1.0

    @property
    def false_positives(self) -> int:
        return self.aabb_hits - self.ellipsoid_hits

    def merge(self, other: "RenderStats"):
        for k in _STAT_KEYS + ("pairs", "composited"):
            setattr(self, k, getattr(self, k) + getattr(other, k))

    def to_dict(self) -> dict:
        d = {k: getattr(self, k) for k in _STAT_KEYS}
        d["false_positives"] = self.false_positives
        return d

    pairs: int = 0
    composited: int = 0

    @classmethod
    def from_counts(cls, counts) -> "RenderStats":
        """From the 10 device counters (gsx_stats)."""
        keys = _STAT_KEYS + ("pairs", "composited")
        return cls(**{k: int(v) for k, v in zip(keys, counts)})


_LAZY_FIELDS = _STAT_KEYS + ("pairs", "composited", "transmittance")


class LazyRenderStats(RenderStats):
    """RenderStats whose counters are gathered only when first read.

    The exact counters need the STATS variant of the forward (every AABB /
    ellipsoid overlap counted per segment, the reference's overflow
    sub-collects emulated): ~15x the plain frame at C3.  `render_image`
    returns this so the drop-in renders at full speed and pays for the
    counters only if the caller looks at them.  `compute()` -> RenderStats
    runs then; it must see the scene unchanged (`scene.version`)."""

    def __init__(self, compute):  # noqa: D107 -- fields materialize lazily
        object.__setattr__(self, "_compute", compute)

    def _materialize(self):
        compute = object.__getattribute__(self, "_compute")
        if compute is not None:
            object.__setattr__(self, "_compute", None)
            s = compute()
            for k in _LAZY_FIELDS:
                object.__setattr__(self, k, getattr(s, k))

    @property
    def ready(self) -> bool:
        return object.__getattribute__(self, "_compute") is None

    def __getattribute__(self, name):
        if name in _LAZY_FIELDS or name == "__dict__":
            object.__getattribute__(self, "_materialize")()
        return object.__getattribute__(self, name)

    def __setattr__(self, name, value):
        if name in _LAZY_FIELDS:
            self._materialize()
        object.__setattr__(self, name, value)


def segment_step(cfg: RenderConfig, d_i: float, t_i: float) -> float:
    """renderer.py:148-157 (host mirror; the kernel evaluates the same formula)."""
    t = max(t_i, cfg.t_eps)
    boost = math.exp(-math.log(t) / 3.0)
    step = min(max(d_i / cfg.beta, cfg.dt_min) * boost, cfg.dt_max)
    return cfg.n_s * step
