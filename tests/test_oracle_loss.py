"""Pin the numpy loss oracle (oracle/loss.py) against the reference's own SSIM /
image-loss values (tests/golden/misc.npz) and finite differences.  CPU only."""

import numpy as np
import pytest

from conftest import golden
from oracle import loss as OL


def test_ssim_and_loss_match_reference_exactly():
    g = golden("misc")
    assert OL.ssim(g["loss.a"], g["loss.b"]) == pytest.approx(float(g["loss.ssim"]), abs=1e-14)
    assert OL.image_loss(g["loss.a"], g["loss.b"]) == pytest.approx(float(g["loss.total"]),
                                                                    abs=1e-14)
    assert OL.ssim(g["loss.g1"], g["loss.g2"]) == pytest.approx(float(g["loss.ssim_gray"]),
                                                               abs=1e-14)


def test_identical_images():
    a = np.random.default_rng(0).uniform(size=(32, 32, 3))
    assert OL.ssim(a, a) == pytest.approx(1.0, abs=1e-12)


@pytest.mark.parametrize("shape", [(14, 13, 3), (11, 17, 3), (20, 20)])
def test_loss_gradient_matches_finite_differences(shape):
    rng = np.random.default_rng(1)
    a = rng.uniform(size=shape)
    b = np.clip(a + rng.normal(0, 0.1, a.shape), 0, 1)
    gr = OL.image_loss_grad(a, b, 0.2)
    fd = np.zeros_like(a)
    h = 1e-6
    for idx in np.ndindex(a.shape):
        ap, am = a.copy(), a.copy()
        ap[idx] += h
        am[idx] -= h
        fd[idx] = (OL.image_loss(ap, b) - OL.image_loss(am, b)) / (2 * h)
    assert np.abs(gr - fd).max() < 1e-6 * np.abs(fd).max()


def test_isotropic_loss_against_reference_formula():
    # geometry.py:193-233; r_max(1,1,10) = 37.9
    assert OL.ratio_upper_bound([1, 1, 10]) == pytest.approx(37.9, abs=0.05)
    assert OL.ratio_upper_bound([1, 1, 1]) == pytest.approx(6 / np.pi, abs=1e-12)
    rng = np.random.default_rng(2)
    s = rng.uniform(0.05, 0.5, size=(50, 3)) * np.array([1, 1, 8.0])
    L, g = OL.isotropic_loss(s, r0=2.0)
    h = 1e-7
    for i in range(5):
        for k in range(3):
            sp, sm = s.copy(), s.copy()
            sp[i, k] += h
            sm[i, k] -= h
            fd = (OL.isotropic_loss(sp, 2.0)[0] - OL.isotropic_loss(sm, 2.0)[0]) / (2 * h)
            assert g[i, k] == pytest.approx(fd, rel=1e-5, abs=1e-9)
