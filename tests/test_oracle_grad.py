"""Pin the oracle's analytic float64 backward (the reference has none) by
central finite differences of the oracle's own forward.  CPU only.

sigma_eps = 1e-8 makes the truncation jump (sigma_eps * dt) negligible and
t_eps = 1e-12 disables early termination, so the rendered functional is smooth
in every record value."""

import numpy as np
import pytest

import oracle as O
from paper_2509_07782_b200.scenes import f32_records, gen_test_scene_records, orbit_poses

GROUPS = {"mean": (0, 3), "quat": (3, 7), "scale": (7, 10), "sigma": (10, 11), "sh": (11, 38),
          "axis": (38, 59), "sharp": (59, 66), "amp": (66, 87)}


@pytest.mark.parametrize("mode", ["uniform", "adaptive"])
def test_oracle_backward_matches_finite_differences(mode):
    rec = f32_records(gen_test_scene_records("random-cloud", count=4, seed=3, anisotropy=2.0,
                                             base_scale=0.25))
    eps = 1e-8
    center, quat = orbit_poses(1, 3.0)[0]
    rays = O.camera_rays(center, quat, 10.0, 6, 6)
    cfg = O.OCfg.make(dt=0.01, t_eps=1e-12, mode=mode, dt_min=0.01, dt_max=0.01)
    rng = np.random.default_rng(0)
    m = rays.shape[0]
    gC, gD, gT = rng.normal(size=(m, 3)), 0.1 * rng.normal(size=m), rng.normal(size=m)
    _, _, _, grad = O.OracleScene(rec, eps).backward_rays(rays, cfg, gC, gD, gT)

    def loss(r):
        R, T, D, _ = O.OracleScene(r, eps).march_rays(rays, cfg, clip=True)
        return float((R * gC).sum() + (D * gD).sum() + (T * gT).sum())

    fd = np.zeros_like(grad)
    for i in range(rec.shape[0]):
        for k in range(87):
            h = 1e-6 * max(abs(rec[i, k]), 1e-2)
            rp, rm = rec.copy(), rec.copy()
            rp[i, k] += h
            rm[i, k] -= h
            fd[i, k] = (loss(rp) - loss(rm)) / (2 * h)
    for g, (a, b) in GROUPS.items():
        num = np.linalg.norm(grad[:, a:b] - fd[:, a:b])
        den = max(np.linalg.norm(fd[:, a:b]), 1e-12)
        assert num / den < 1e-5, (g, num / den)
