"""Golden vectors for the host geometry / appearance value helpers, from the
REFERENCE (geometry.py:67-233, appearance.py:26-98).

Run in the build container only (imports /root/reference/pkg/src):

    python tests/golden/make_golden_geometry.py

Writes geometry.npz: 60 random shapes (mean, quat, scales incl. some below
S_MIN, sigma) with their iso_scale, aabb_of, ellipsoid_volume, volume_ratio,
ratio_upper_bound and its gradient at sigma_eps = 0.01, the isotropic_loss
of the list at r0 = 3, and eval_radiance of 40 random appearance records at
random directions.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from gsray.appearance import AppearanceCoeffs, eval_radiance  # noqa: E402
from gsray.geometry import (GaussianShape, IsoLossConfig, aabb_of, ellipsoid_volume,  # noqa: E402
                            iso_scale, isotropic_loss, ratio_upper_bound,
                            ratio_upper_bound_gradient, volume_ratio)


def main():
    rng = np.random.default_rng(17)
    n = 60
    means = rng.uniform(-2, 2, (n, 3))
    quats = rng.normal(size=(n, 4))
    scales = 10.0 ** rng.uniform(-3, 0, (n, 3))
    scales[::17, 1] = 1e-9  # clamped to S_MIN
    sigmas = rng.uniform(0.05, 5.0, n)
    shapes = [GaussianShape(m, q, s, float(g)) for m, q, s, g in zip(means, quats, scales, sigmas)]
    out = {"means": means, "quats": quats, "scales": scales, "sigmas": sigmas,
           "iso": np.array([iso_scale(s, 0.01) for s in shapes]),
           "aabb_lo": np.array([aabb_of(s, 0.01).lo for s in shapes]),
           "aabb_hi": np.array([aabb_of(s, 0.01).hi for s in shapes]),
           "vol": np.array([ellipsoid_volume(s, 0.01) for s in shapes]),
           "ratio": np.array([volume_ratio(s) for s in shapes]),
           "rmax": np.array([ratio_upper_bound(s.scales) for s in shapes]),
           "rmax_grad": np.array([ratio_upper_bound_gradient(s.scales) for s in shapes])}
    ls, g = isotropic_loss(shapes, IsoLossConfig(r0=3.0))
    out["iso_loss"], out["iso_grad"] = np.array(ls), g
    recs, dirs, rad = [], [], []
    for _ in range(40):
        c = AppearanceCoeffs(rng.normal(size=(9, 3)), rng.normal(size=(7, 3)),
                             rng.uniform(0, 20, 7), rng.normal(size=(7, 3)))
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        recs.append(np.concatenate([c.sh.ravel(), c.sg_axis.ravel(), c.sg_sharp,
                                    c.sg_amp.ravel()]))
        dirs.append(d)
        rad.append(eval_radiance(c, d))
    out["app"], out["app_dirs"], out["app_rgb"] = np.array(recs), np.array(dirs), np.array(rad)
    np.savez_compressed(OUT / "geometry.npz", **out)
    print("wrote", OUT / "geometry.npz")


if __name__ == "__main__":
    main()
