"""Synthetic inputs: procedural scenes as 87-float records and orbit cameras.

Host-side numpy; produces the `.gsx` record layout (scene_io.py:26-44):
mean[0:3] quat(w,x,y,z)[3:7] scales[7:10] sigma~[10] sh 9x3 [11:38]
sg_axis 7x3 [38:59] sg_sharp 7 [59:66] sg_amp 7x3 [66:87].

`gen_test_scene_records` reproduces the reference generator
`gen_test_scene` (scene_io.py:206-273, `_random_appearance` :193-203) draw for
draw, so the same seed yields the same float64 records (checked against the
reference in tests/golden).  `synth_records` is the vectorised generator for
the large benchmark configs (same distributions, different stream).
"""

from __future__ import annotations

import math

import numpy as np

NREC = 87
N_SH = 9
N_SG = 7
S_MIN = 1e-7
_C0 = 0.5 * math.sqrt(1.0 / math.pi)


def _normalize_record(rec: np.ndarray) -> np.ndarray:
    """What a record looks like after GaussianShape/AppearanceCoeffs ingestion
    (geometry.py:77-87, appearance.py:62-76): unit quaternion, scales clamped at
    S_MIN, unit SG axes.  Works on (N, 87)."""
    rec = np.array(rec, dtype=np.float64, copy=True).reshape(-1, NREC)
    q = rec[:, 3:7]
    rec[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    rec[:, 7:10] = np.maximum(rec[:, 7:10], S_MIN)
    ax = rec[:, 38:59].reshape(-1, N_SG, 3)
    rec[:, 38:59] = (ax / np.linalg.norm(ax, axis=2, keepdims=True)).reshape(-1, 21)
    return rec


def _appearance_record(rng: np.random.Generator) -> np.ndarray:
    """scene_io.py:193-203 _random_appearance, same draw order."""
    rgb = rng.uniform(0.2, 0.8, size=3)
    sh = np.zeros((N_SH, 3))
    sh[0] = rgb / _C0
    sh[1:] = rng.uniform(-0.1, 0.1, size=(N_SH - 1, 3))
    axes = rng.standard_normal((N_SG, 3))
    axes = axes / np.linalg.norm(axes, axis=1)[:, None]  # appearance.py:64-68
    sharp = rng.uniform(0.0, 20.0, size=N_SG)
    amp = rng.uniform(0.0, 0.15, size=(N_SG, 3))
    return np.concatenate([sh.ravel(), axes.ravel(), sharp, amp.ravel()])


def gen_test_scene_records(kind: str = "random-cloud", count: int = 32, seed: int = 0,
                           anisotropy: float = 1.0, extent: float = 1.0,
                           base_scale: float = 0.08) -> np.ndarray:
    """(N, 87) float64 records equal to the reference's gen_test_scene output
    after ingestion (normalized quaternions / axes)."""
    rng = np.random.default_rng(seed)
    recs = []

    def shape(mean, quat, scales, sigma):
        # GaussianShape.__post_init__ (geometry.py:78-81): 1-D norm, clamp
        quat = np.asarray(quat, dtype=float).reshape(4)
        quat = quat / np.linalg.norm(quat)
        scales = np.maximum(np.asarray(scales, dtype=float).reshape(3), S_MIN)
        return np.concatenate([np.asarray(mean, float), quat, scales, [float(sigma)]])

    if kind in ("single-gaussian", "single"):
        s = shape(np.zeros(3), [1, 0, 0, 0], np.full(3, base_scale), 2.0)
        recs.append(np.concatenate([s, _appearance_record(rng)]))
    elif kind == "grid":
        side = max(int(round(count ** (1.0 / 3.0))), 1)
        xs = np.linspace(-extent, extent, side) if side > 1 else np.array([0.0])
        for ix in xs:
            for iy in xs:
                for iz in xs:
                    sig = float(rng.uniform(1.0, 4.0))
                    s = shape([ix, iy, iz], [1, 0, 0, 0], np.full(3, base_scale), sig)
                    recs.append(np.concatenate([s, _appearance_record(rng)]))
    elif kind == "random-cloud":
        for _ in range(count):
            q = rng.standard_normal(4)
            b = base_scale * rng.uniform(0.6, 1.4)
            mean = rng.uniform(-extent, extent, size=3)
            sig = float(rng.uniform(1.0, 4.0))
            s = shape(mean, q, np.array([b, b, b * anisotropy]), sig)
            recs.append(np.concatenate([s, _appearance_record(rng)]))
    elif kind == "shell":
        for _ in range(count):
            u = rng.standard_normal(3)
            u = u / np.linalg.norm(u)
            q = rng.standard_normal(4)
            sig = float(rng.uniform(1.0, 4.0))
            s = shape(extent * u, q, np.full(3, base_scale), sig)
            recs.append(np.concatenate([s, _appearance_record(rng)]))
    else:
        raise ValueError(f"unknown scene kind {kind!r}")
    return np.stack(recs)


def f32_records(rec: np.ndarray) -> np.ndarray:
    """Round records to float32 (the .gsx wire format, scene_io.py:44) and back to
    float64, so host, oracle and device see identical values."""
    return np.asarray(rec, dtype=np.float32).astype(np.float64)


def _random_appearance_block(rng: np.random.Generator, n: int) -> np.ndarray:
    rgb = rng.uniform(0.2, 0.8, size=(n, 3))
    sh = np.empty((n, N_SH, 3))
    sh[:, 0] = rgb / _C0
    sh[:, 1:] = rng.uniform(-0.1, 0.1, size=(n, N_SH - 1, 3))
    axes = rng.standard_normal((n, N_SG, 3))
    sharp = rng.uniform(0.0, 20.0, size=(n, N_SG))
    amp = rng.uniform(0.0, 0.15, size=(n, N_SG, 3))
    return np.concatenate([sh.reshape(n, -1), axes.reshape(n, -1), sharp,
                           amp.reshape(n, -1)], axis=1)


def synth_records(kind: str, count: int, seed: int = 0, anisotropy: float = 1.0,
                  extent: float = 1.0, base_scale: float | None = None,
                  sigma_scale: float | None = None, r_max_bound: float | None = None,
                  shell_fraction: float = 0.0, shell_radius=(10.0, 50.0),
                  view_radius: float = 3.5) -> np.ndarray:
    """Vectorised large-N generator (float32-representable float64 records).

    Defaults follow SURVEY.md 8(d): base = 0.08 * (32/N)^(1/3) and
    sigma~ scaled by 0.08/base so per-primitive optical depth stays in the
    reference's range.  `r_max_bound` clamps the anisotropy so that
    ratio_upper_bound((1,1,a)) <= r_max_bound (the paper's volume-ratio bound,
    geometry.py:193-202).  `shell_fraction` of the primitives are placed on a
    background shell with radius in `shell_radius` and scale proportional to
    distance (the Mip-NeRF360-shaped C3/C4 scenes).
    """
    rng = np.random.default_rng(seed)
    n = int(count)
    if base_scale is None:
        base_scale = 0.08 * (32.0 / max(n, 1)) ** (1.0 / 3.0)
    if sigma_scale is None:
        sigma_scale = 0.08 / base_scale
    a = float(anisotropy)
    if r_max_bound is not None:
        a = min(a, max_anisotropy_for_bound(r_max_bound))
    n_shell = int(round(shell_fraction * n))
    n_in = n - n_shell
    rec = np.empty((n, NREC))
    q = rng.standard_normal((n, 4))
    b = base_scale * rng.uniform(0.6, 1.4, size=n)
    if kind == "random-cloud":
        mean_in = rng.uniform(-extent, extent, size=(n_in, 3))
    elif kind == "ball":
        v = rng.standard_normal((n_in, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        r = extent * rng.uniform(0, 1, size=(n_in, 1)) ** (1.0 / 3.0)
        mean_in = v * r
    elif kind == "shell":
        v = rng.standard_normal((n_in, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        mean_in = extent * v
    elif kind == "surface":
        # closed surface-like object: shell plus a thin interior cloud
        v = rng.standard_normal((n_in, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        r = extent * (1.0 - 0.15 * rng.uniform(0, 1, size=(n_in, 1)) ** 3)
        mean_in = v * r
    else:
        raise ValueError(f"unknown scene kind {kind!r}")
    means = np.empty((n, 3))
    means[:n_in] = mean_in
    scale_mul = np.ones(n)
    if n_shell:
        v = rng.standard_normal((n_shell, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        rad = rng.uniform(shell_radius[0], shell_radius[1], size=n_shell)
        means[n_in:] = v * rad[:, None]
        # same angular size as a foreground primitive seen from `view_radius`
        scale_mul[n_in:] = rad / view_radius
    rec[:, 0:3] = means
    rec[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    bb = b * scale_mul
    rec[:, 7] = bb
    rec[:, 8] = bb
    rec[:, 9] = bb * a
    sig = rng.uniform(1.0, 4.0, size=n) * sigma_scale
    if n_shell:
        # keep background optical depth comparable: density ~ 1/size
        sig[n_in:] /= scale_mul[n_in:]
        sig = np.maximum(sig, 0.02)
    rec[:, 10] = sig
    rec[:, 11:] = _random_appearance_block(rng, n)
    rec = _normalize_record(rec)
    return f32_records(rec)


def ratio_upper_bound(scales) -> float:
    """geometry.py:193-202."""
    s = np.maximum(np.asarray(scales, dtype=float).reshape(3), S_MIN)
    return (2.0 / (math.pi * math.sqrt(3.0))) * float(np.sum(s ** 2) ** 1.5 / np.prod(s))


def max_anisotropy_for_bound(r0: float) -> float:
    """Largest a with ratio_upper_bound((1,1,a)) <= r0 (bisection; monotone for a>=1)."""
    lo, hi = 1.0, 1e6
    if ratio_upper_bound((1, 1, 1)) > r0:
        return 1.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if ratio_upper_bound((1, 1, mid)) <= r0:
            lo = mid
        else:
            hi = mid
    return lo


# -- cameras (scene_io.py:158-187, geometry.py:45-64) -------------------------

def rotation_to_quat(r: np.ndarray) -> np.ndarray:
    """Scalar-first unit quaternion (Shepperd), geometry.py:45-64."""
    r = np.asarray(r, dtype=float)
    t = np.trace(r)
    if t > 0:
        s = math.sqrt(t + 1.0) * 2.0
        q = np.array([0.25 * s, (r[2, 1] - r[1, 2]) / s, (r[0, 2] - r[2, 0]) / s,
                      (r[1, 0] - r[0, 1]) / s])
    else:
        i = int(np.argmax(np.diag(r)))
        j, k = (i + 1) % 3, (i + 2) % 3
        s = math.sqrt(1.0 + r[i, i] - r[j, j] - r[k, k]) * 2.0
        q = np.empty(4)
        q[0] = (r[k, j] - r[j, k]) / s
        q[1 + i] = 0.25 * s
        q[1 + j] = (r[j, i] + r[i, j]) / s
        q[1 + k] = (r[k, i] + r[i, k]) / s
    return q / np.linalg.norm(q)


def look_at(center, target, up=(0.0, 1.0, 0.0)):
    """(center, quat) of a camera looking at target, +z forward, +y down."""
    center = np.asarray(center, dtype=float)
    fwd = np.asarray(target, dtype=float) - center
    fwd = fwd / np.linalg.norm(fwd)
    up = np.asarray(up, dtype=float)
    right = np.cross(fwd, up)
    if np.linalg.norm(right) < 1e-9:
        right = np.cross(fwd, [1.0, 0.0, 0.0])
    right = right / np.linalg.norm(right)
    down = np.cross(fwd, right)
    rot = np.stack([right, down, fwd], axis=1)
    return center, rotation_to_quat(rot)


def orbit_poses(n: int, radius: float, elevation: float = 0.35, target=(0.0, 0.0, 0.0)):
    """scene_io.py:175-187: n (center, quat) poses on a circle around target."""
    out = []
    target = np.asarray(target, dtype=float)
    for i in range(n):
        a = 2.0 * math.pi * i / n
        center = target + radius * np.array([math.cos(a) * math.cos(elevation),
                                             math.sin(elevation),
                                             math.sin(a) * math.cos(elevation)])
        out.append(look_at(center, target))
    return out
