"""float64 numpy restatement of the reference image loss (densify.py:99-153)
and of its gradient w.r.t. the rendered image -- TEST INFRASTRUCTURE ONLY.

SSIM statistics use an 11-tap Gaussian (sigma 1.5, truncate 3.5 -> radius 5)
applied separably with scipy's 'reflect' boundary (numpy 'symmetric' padding:
d c b a | a b c d), K1 = 0.01, K2 = 0.03, data range 1, 5-px crop, mean over
channels (densify.py:106-132).  Pinned against the reference's values in
tests/golden/misc.npz and against finite differences (tests/test_oracle_loss.py).
"""

from __future__ import annotations

import math

import numpy as np

R = 5


def taps():
    i = np.arange(-R, R + 1, dtype=np.float64)
    w = np.exp(-0.5 * i * i / (1.5 * 1.5))
    return w / w.sum()


def _filt1d(a, axis):
    w = taps()
    pad = [(0, 0)] * a.ndim
    pad[axis] = (R, R)
    ap = np.pad(a, pad, mode="symmetric")
    n = a.shape[axis]
    out = np.zeros_like(a)
    for k in range(-R, R + 1):
        sl = [slice(None)] * a.ndim
        sl[axis] = slice(R + k, R + k + n)
        out += w[k + R] * ap[tuple(sl)]
    return out


def _filt1d_T(g, axis):
    """Adjoint of _filt1d (transpose of symmetric padding + correlation)."""
    w = taps()
    n = g.shape[axis]
    shape = list(g.shape)
    shape[axis] = n + 2 * R
    gp = np.zeros(shape)
    for k in range(-R, R + 1):
        sl = [slice(None)] * g.ndim
        sl[axis] = slice(R + k, R + k + n)
        gp[tuple(sl)] += w[k + R] * g

    def take(lo, hi):
        sl = [slice(None)] * g.ndim
        sl[axis] = slice(lo, hi)
        return gp[tuple(sl)]

    out = take(R, R + n).copy()
    # fold the padded margins back onto their (symmetric) sources
    left = np.flip(take(0, R), axis=axis)      # pad index R-1-m -> x[m]
    right = np.flip(take(R + n, n + 2 * R), axis=axis)  # pad index R+n+m -> x[n-1-m]
    sl = [slice(None)] * g.ndim
    sl[axis] = slice(0, R)
    out[tuple(sl)] += left
    sl[axis] = slice(n - R, n)
    out[tuple(sl)] += right
    return out


def gfilt(img):
    """gaussian_filter(img, 1.5, truncate=3.5) on a 2-D array (axis 0 then 1)."""
    return _filt1d(_filt1d(img, 0), 1)


def gfilt_T(g):
    return _filt1d_T(_filt1d_T(g, 1), 0)


def ssim(a, b):
    """densify.py:99-132 _ssim."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.ndim == 2:
        a, b = a[..., None], b[..., None]
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    vals = []
    for ch in range(a.shape[2]):
        x, y = a[..., ch], b[..., ch]
        ux, uy = gfilt(x), gfilt(y)
        vx = gfilt(x * x) - ux * ux
        vy = gfilt(y * y) - uy * uy
        cov = gfilt(x * y) - ux * uy
        s = ((2 * ux * uy + c1) * (2 * cov + c2)) / ((ux * ux + uy * uy + c1) * (vx + vy + c2))
        vals.append(s[R:-R, R:-R].mean())
    return float(np.mean(vals))


def image_loss(rendered, target, mix=0.2, lambda_s=0.0, iso_loss=0.0):
    """densify.py:139-153 image_loss."""
    r = np.asarray(rendered, np.float64)
    t = np.asarray(target, np.float64)
    l1 = float(np.mean(np.abs(r - t)))
    total = (1.0 - mix) * l1
    if mix > 0.0:
        total += mix * (1.0 - ssim(r, t)) / 2.0
    return total + lambda_s * iso_loss


def image_loss_grad(rendered, target, mix=0.2):
    """Analytic dL/d rendered for image_loss (float64)."""
    r = np.asarray(rendered, np.float64)
    t = np.asarray(target, np.float64)
    squeeze = r.ndim == 2
    if squeeze:
        r, t = r[..., None], t[..., None]
    H, W, C = r.shape
    g = (1.0 - mix) * np.sign(r - t) / r.size
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    n_crop = (H - 2 * R) * (W - 2 * R) * C
    for ch in range(C):
        x, y = r[..., ch], t[..., ch]
        ux, uy = gfilt(x), gfilt(y)
        vx = gfilt(x * x) - ux * ux
        vy = gfilt(y * y) - uy * uy
        cov = gfilt(x * y) - ux * uy
        A1, B1 = 2 * ux * uy + c1, 2 * cov + c2
        A2, B2 = ux * ux + uy * uy + c1, vx + vy + c2
        D = A2 * B2
        S = A1 * B1 / D
        mask = np.zeros_like(S)
        mask[R:-R, R:-R] = 1.0
        a = mask * (2 * uy * (B1 - A1) - S * 2 * ux * (B2 - A2)) / D
        b = mask * (-S / B2)
        c = mask * (2 * A1 / D)
        gs = gfilt_T(a) + 2 * x * gfilt_T(b) + y * gfilt_T(c)
        g[..., ch] += -0.5 * mix / n_crop * gs
    return g[..., 0] if squeeze else g


def ratio_upper_bound(s):
    """geometry.py:193-202."""
    s = np.maximum(np.asarray(s, np.float64), 1e-7)
    return (2.0 / (math.pi * math.sqrt(3.0))) * np.sum(s ** 2, -1) ** 1.5 / np.prod(s, -1)


def isotropic_loss(scales, r0=10.0):
    """geometry.py:215-233: (L_s, dL_s/ds (N,3)) for raw (N,3) scales."""
    raw = np.asarray(scales, np.float64).reshape(-1, 3)
    s = np.maximum(raw, 1e-7)
    n = s.shape[0]
    r = ratio_upper_bound(s)
    act = r > r0
    ss = np.sum(s ** 2, 1, keepdims=True)
    g = r[:, None] * (3.0 * s / ss - 1.0 / s) / n
    g = np.where(act[:, None] & (raw > 1e-7), g, 0.0)
    return float(np.sum(np.where(act, r - r0, 0.0)) / n), g
