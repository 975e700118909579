"""Pin the densification statistics chain against the reference's own
observe_scene (densify.py:190-204) accumulators in tests/golden/densify.npz
(tests/golden/make_golden_densify.py).  CPU only.

The reference finite-differences the loss with step h = 1e-4 x the scene
diagonal (densify.py:178-179).  At that step a sample can cross a
primitive's truncation boundary, where the density jumps from sigma_eps to
0, so the reference's FD norm includes that jump; the analytic gradient of
the truncated model (and FD with a smaller step) does not.  Hence two pins:
  1. the oracle's FD at the reference's own step reproduces the reference's
     accumulators (same forward, same loss, same differencing);
  2. the oracle's analytic backward equals its FD at h/100 (no crossing),
     which is what the GPU observation reproduces (test_gpu_densify.py), to
     5e-3: the analytic gradient holds sample positions fixed, while moving a
     primitive that defines the scene bounds also moves the clipped t_n
     that anchors every ray's sample grid (renderer.py:160-175) -- FD sees
     that (primitive 1 here: 2e-4 with L1, 4e-3 with DSSIM)."""

import numpy as np
import pytest

import oracle as O
from conftest import golden
from oracle import loss as OL


def _setup():
    g = golden("densify")
    w, h = int(g["cam.cam_w"]), int(g["cam.cam_h"])
    rays = O.camera_rays(g["cam.cam_center"], g["cam.cam_quat"], float(g["cam.cam_focal"]), w, h)
    return g, rays, w, h, O.OCfg.make(dt=0.02)


def _loss(rec, rays, cfg, target, mix, w, h):
    R, _, _, _ = O.OracleScene(rec, 0.01).march_rays(rays, cfg)
    return OL.image_loss(R.reshape(h, w, 3), target, mix)


def _fd_norms(g, rays, cfg, mix, w, h, step_scale):
    rec = g["records"]
    osc = O.OracleScene(rec, 0.01)
    step = 1e-4 * np.linalg.norm(osc.bounds_hi - osc.bounds_lo) * step_scale
    out = []
    for i in range(len(rec)):
        gr = np.zeros(3)
        for a in range(3):
            rp, rm = rec.copy(), rec.copy()
            rp[i, a] += step
            rm[i, a] -= step
            gr[a] = (_loss(rp, rays, cfg, g["target"], mix, w, h) -
                     _loss(rm, rays, cfg, g["target"], mix, w, h)) / (2 * step)
        out.append(np.linalg.norm(gr))
    return np.array(out)


@pytest.mark.parametrize("li", [0, 1])
def test_oracle_fd_reproduces_reference_accumulators(li):
    g, rays, w, h, cfg = _setup()
    mix = float(g[f"mix{li}"])
    norms = _fd_norms(g, rays, cfg, mix, w, h, 1.0)
    rec = g["records"]
    alpha = np.linalg.norm(rec[:, 0:3] - g["cam.cam_center"], axis=1) / float(g["cam.cam_focal"])
    np.testing.assert_allclose(norms, g[f"sum_raw{li}"], rtol=1e-6)
    np.testing.assert_allclose(alpha * norms, g[f"sum_weighted{li}"], rtol=1e-6)
    assert g[f"counts{li}"].tolist() == [1] * len(rec)


@pytest.mark.parametrize("li", [0, 1])
def test_oracle_analytic_equals_small_step_fd(li):
    g, rays, w, h, cfg = _setup()
    mix = float(g[f"mix{li}"])
    osc = O.OracleScene(g["records"], 0.01)
    R, _, _, _ = osc.march_rays(rays, cfg)
    gI = OL.image_loss_grad(R.reshape(h, w, 3), g["target"], mix)
    _, _, _, grad = osc.backward_rays(rays, cfg, gI.reshape(-1, 3), np.zeros(h * w),
                                      np.zeros(h * w))
    analytic = np.linalg.norm(grad[:, 0:3], axis=1)
    np.testing.assert_allclose(analytic, _fd_norms(g, rays, cfg, mix, w, h, 1e-2), rtol=5e-3)
