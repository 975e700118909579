"""The dense oracles (oracle/gsray_oracle.c: reference_integrate /
reference_render renderer.py:440-493, eval_fields appearance.py:107-134)
against golden vectors the reference itself produced
(tests/golden/make_golden_dense.py -> dense.npz)."""

import numpy as np

import oracle as O
from conftest import golden


def _scene(g):
    return O.OracleScene(g["rec"], 0.01)


def test_reference_render_matches_reference():
    g = golden("dense")
    osc = _scene(g)
    W, H = (int(v) for v in g["cam_wh"])
    rays = O.camera_rays(g["cam_center"], g["cam_quat"], float(g["cam_focal"]), W, H)
    img = osc.reference_rays(rays, 0.0025 / 8.0, clip=True, threads=4).reshape(H, W, 3)
    np.testing.assert_allclose(img, g["ref_img"], rtol=0, atol=1e-12)
    assert img.max() > 0.05  # the view sees the Gaussians


def test_reference_integrate_matches_reference():
    g = golden("dense")
    out = _scene(g).reference_rays(g["int_rays"], 0.001, background=g["int_bg"], clip=False)
    np.testing.assert_allclose(out, g["int_rgb"], rtol=0, atol=1e-12)


def test_eval_fields_matches_reference():
    g = golden("dense")
    osc = _scene(g)
    for key, active in (("all", None), ("a02", [2, 0]), ("a134", [1, 3, 4])):
        got = [osc.eval_fields(x, d, active) for x, d in zip(g["f_pts"], g["f_dirs"])]
        sig = np.array([s for s, _ in got])
        col = np.array([c for _, c in got])
        np.testing.assert_allclose(sig, g[f"f_sigma_{key}"], rtol=1e-12, atol=0)
        np.testing.assert_allclose(col, g[f"f_color_{key}"], rtol=0, atol=1e-12)
    assert (g["f_sigma_all"] > 0).sum() > 20 and (g["f_sigma_all"] == 0).sum() > 5


def test_march_vs_dense_psnr_oracle():
    """test_acceptance.py:122-131 on the oracle: the uniform march of the
    5-Gaussian view is within 45 dB of its dt/8 dense quadrature."""
    g = golden("dense")
    ref, img = g["ref_img"], g["march_img"]
    mse = np.mean((ref - img) ** 2)
    assert 10 * np.log10(1.0 / mse) >= 45.0
