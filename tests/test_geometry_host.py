"""Host value helpers (geometry.py / appearance.py of the drop-in package)
against golden vectors the reference produced
(tests/golden/make_golden_geometry.py -> geometry.npz)."""

import numpy as np
import pytest

from conftest import golden


def test_shape_geometry_matches_reference():
    import paper_2509_07782_b200 as G
    from paper_2509_07782_b200.geometry import ratio_upper_bound_gradient

    g = golden("geometry")
    shapes = [G.GaussianShape(m, q, s, float(x))
              for m, q, s, x in zip(g["means"], g["quats"], g["scales"], g["sigmas"])]
    tol = dict(rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose([G.iso_scale(s, 0.01) for s in shapes], g["iso"], **tol)
    np.testing.assert_allclose([G.aabb_of(s, 0.01).lo for s in shapes], g["aabb_lo"], **tol)
    np.testing.assert_allclose([G.aabb_of(s, 0.01).hi for s in shapes], g["aabb_hi"], **tol)
    np.testing.assert_allclose([G.ellipsoid_volume(s, 0.01) for s in shapes], g["vol"], **tol)
    np.testing.assert_allclose([G.volume_ratio(s) for s in shapes], g["ratio"], **tol)
    np.testing.assert_allclose([G.ratio_upper_bound(s.scales) for s in shapes], g["rmax"], **tol)
    np.testing.assert_allclose([ratio_upper_bound_gradient(s.scales) for s in shapes],
                               g["rmax_grad"], **tol)


def test_shape_validation():
    import paper_2509_07782_b200 as G

    with pytest.raises(ValueError):
        G.GaussianShape([0, 0, 0], [1, 0, 0, 0], [1, 1, 1], -1.0)
    s = G.GaussianShape([0, 0, 0], [2, 0, 0, 0], [0, 1, 1], 0.005)
    assert s.scales[0] == 1e-7 and np.allclose(s.quat, [1, 0, 0, 0])
    with pytest.raises(G.EmptyIsosurface):
        G.iso_scale(s, 0.01)
    with pytest.raises(ValueError):
        G.Aabb([1, 0, 0], [0, 1, 1])
    with pytest.raises(ValueError):
        G.IsoLossConfig(r0=1.0)


def test_eval_radiance_matches_reference():
    import paper_2509_07782_b200 as G

    g = golden("geometry")
    for rec, d, want in zip(g["app"], g["app_dirs"], g["app_rgb"]):
        c = G.AppearanceCoeffs(rec[:27], rec[27:48], rec[48:55], rec[55:76])
        np.testing.assert_allclose(G.eval_radiance(c, d), want, rtol=1e-12, atol=1e-13)
    k = G.AppearanceCoeffs.constant([0.25, 0.5, 1.0])
    np.testing.assert_allclose(G.eval_radiance(k, [0.6, 0.0, 0.8]), [0.25, 0.5, 1.0])
    with pytest.raises(ValueError):
        G.AppearanceCoeffs(np.zeros((9, 3)), np.zeros((7, 3)), np.zeros(7), np.zeros((7, 3)))
