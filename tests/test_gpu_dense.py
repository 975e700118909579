"""Device dense oracles (csrc/dense.cu: reference_integrate / reference_render
renderer.py:440-493, eval_fields appearance.py:107-134) against the float64
oracle on the same float32 records, against the reference's own golden
vectors (dense.npz, whose records are float64: agreement to the float32
rounding of the records), and the reference tests that use them:

* the renderer-correctness acceptance criterion (test_acceptance.py:102-133):
  the 64x64 5-Gaussian render_image within 45 dB PSNR of its dt/8 dense
  quadrature -- both on the device;
* the mixture-field tests of test_appearance.py:102-143 (truncation, density
  formula to 1e-12, density-weighted colour, `active` order and supersets).
"""

import math

import numpy as np
import pytest

import oracle as O
from conftest import golden
from paper_2509_07782_b200.scenes import f32_records

pytestmark = pytest.mark.gpu


def _golden_scene(G):
    g = golden("dense")
    rec = f32_records(g["rec"])
    cam = G.Camera(center=g["cam_center"], quat=g["cam_quat"], focal=float(g["cam_focal"]),
                   width=int(g["cam_wh"][0]), height=int(g["cam_wh"][1]))
    return g, rec, G.Scene.from_records(rec), O.OracleScene(rec, 0.01), cam


def test_reference_render_vs_oracle_and_reference():
    import paper_2509_07782_b200 as G

    g, rec, scene, osc, cam = _golden_scene(G)
    img = G.reference_render(scene, cam, 0.0025 / 8.0)
    rays = O.camera_rays(cam.center, cam.quat, cam.focal, cam.width, cam.height)
    want = osc.reference_rays(rays, 0.0025 / 8.0, clip=True, threads=8).reshape(img.shape)
    assert np.abs(img - want).max() < 1e-10
    assert np.abs(img - g["ref_img"]).max() < 1e-5  # float32 records vs float64
    assert img.max() > 0.05


def test_reference_integrate_vs_oracle():
    import paper_2509_07782_b200 as G

    g, rec, scene, osc, cam = _golden_scene(G)
    got = G.reference_rays(scene, g["int_rays"], 0.001, background=g["int_bg"])
    want = osc.reference_rays(g["int_rays"], 0.001, background=g["int_bg"])
    assert np.abs(got - want).max() < 1e-10
    assert np.abs(got - g["int_rgb"]).max() < 1e-5
    one = G.reference_integrate(scene, G.Ray(g["int_rays"][3, :3], g["int_rays"][3, 3:6],
                                             g["int_rays"][3, 6], g["int_rays"][3, 7]),
                                0.001, background=g["int_bg"])
    assert np.abs(one - want[3]).max() < 1e-10


def test_eval_fields_vs_oracle_and_reference():
    import paper_2509_07782_b200 as G

    g, rec, scene, osc, cam = _golden_scene(G)
    inv = np.argsort(scene.uids)  # original index -> storage position
    for key, active in (("all", None), ("a02", [2, 0]), ("a134", [1, 3, 4])):
        act = None if active is None else inv[np.asarray(active)]
        sig, col = G.eval_fields_batch(scene, g["f_pts"], g["f_dirs"], act)
        want = [osc.eval_fields(x, d, active) for x, d in zip(g["f_pts"], g["f_dirs"])]
        np.testing.assert_allclose(sig, [s for s, _ in want], rtol=1e-12, atol=1e-300)
        np.testing.assert_allclose(col, [c for _, c in want], rtol=0, atol=1e-12)
        np.testing.assert_allclose(sig, g[f"f_sigma_{key}"], rtol=1e-5, atol=0)


def _two_primitive_scene(G):
    # test_appearance.py:90-99 with float32-exact values (0.25 for 0.3, 0.25 for 0.2)
    shapes = [G.GaussianShape([0, 0, 0], [1, 0, 0, 0], [0.25, 0.25, 0.25], 2.0),
              G.GaussianShape([0.25, 0, 0], [1, 0, 0, 0], [0.25, 0.25, 0.25], 1.0)]
    coeffs = [G.AppearanceCoeffs.constant([1, 0, 0]), G.AppearanceCoeffs.constant([0, 1, 0])]
    return shapes, G.Scene(shapes, coeffs, sigma_eps=0.01)


def test_fields_truncation_and_formula():
    """test_appearance.py:103-119."""
    import paper_2509_07782_b200 as G

    shapes, scene = _two_primitive_scene(G)
    r = G.iso_scale(shapes[0], 0.01)[0]
    inside = G.eval_fields(scene, [0, 0, 0.99 * r], [0, 0, 1])
    outside = G.eval_fields(scene, [0, 0, 3 * r], [0, 0, 1])
    assert inside.sigma > 0
    assert outside.sigma == 0.0 and np.all(outside.color == 0.0)
    s = shapes[0]
    x = np.array([0.0, 0.0, 0.1])
    got = G.eval_fields(scene, x, [0, 0, 1], active=[0])
    y = (x - s.mean) / s.scales
    assert got.sigma == pytest.approx(s.sigma * math.exp(-0.5 * y @ y), rel=1e-12)


def test_fields_weighted_color_and_active():
    """test_appearance.py:121-143."""
    import paper_2509_07782_b200 as G

    _, scene = _two_primitive_scene(G)
    x = np.array([0.1, 0.0, 0.0])
    fs = G.eval_fields(scene, x, [0, 0, 1])
    d0 = G.eval_fields(scene, x, [0, 0, 1], active=[0]).sigma
    d1 = G.eval_fields(scene, x, [0, 0, 1], active=[1]).sigma
    assert fs.sigma == pytest.approx(d0 + d1, rel=1e-12)
    want = (d0 * np.array([1, 0, 0]) + d1 * np.array([0, 1, 0])) / (d0 + d1)
    assert np.allclose(fs.color, want, atol=1e-12)
    a = G.eval_fields(scene, x, [0, 0, 1], active=[0, 1])
    b = G.eval_fields(scene, x, [0, 0, 1], active=[1, 0])
    assert a.sigma == pytest.approx(b.sigma, rel=1e-15) and np.allclose(a.color, b.color,
                                                                         atol=1e-15)
    assert fs.sigma == pytest.approx(a.sigma, rel=1e-15)
    with pytest.raises(ValueError):
        G.eval_fields(scene, x, [0, 0, 1], active=[0, 7])


def test_acceptance_renderer_psnr_45db():
    """test_acceptance.py:122-131: the 64x64 five-Gaussian image of the
    default uniform config within 45 dB of the dt/8 dense reference."""
    import paper_2509_07782_b200 as G

    five = G.gen_test_scene("random-cloud", count=5, seed=42, anisotropy=2.0)
    cam = G.orbit_cameras(1, radius=3.0, focal=64.0, width=64, height=64)[0]
    cfg = G.RenderConfig()
    img, _ = G.render_image(five, cam, cfg)
    ref = G.reference_render(five, cam, cfg.dt / 8.0)
    assert ref.max() > 0.05
    assert G.psnr(img, ref) >= 45.0


def test_march_image_vs_reference_golden():
    import paper_2509_07782_b200 as G

    g, rec, scene, osc, cam = _golden_scene(G)
    img, _ = G.render_image(scene, cam, G.RenderConfig())
    assert np.abs(img - g["march_img"]).max() < 1e-4


def test_isotropic_loss_list_form_vs_reference():
    """geometry.py:215-233 called with a list of shapes (the reference's
    form), evaluated by the device kernel."""
    import paper_2509_07782_b200 as G

    g = golden("geometry")
    shapes = [G.GaussianShape(m, q, s, float(x))
              for m, q, s, x in zip(g["means"], g["quats"], g["scales"], g["sigmas"])]
    val, grad = G.isotropic_loss(shapes, G.IsoLossConfig(r0=3.0))
    assert val == pytest.approx(float(g["iso_loss"]), rel=1e-6)
    big = np.abs(g["iso_grad"]) > 0
    np.testing.assert_allclose(grad[big], g["iso_grad"][big], rtol=1e-5)


def test_deep_tree_traversals_agree():
    """A degenerate, deep LBVH: 3000 primitives at one point
    (identical Morton codes: Karras splits by index) inside a 200-level
    geometric cluster (0.9^k offsets: one code prefix level per primitive
    until the 21-bit grid saturates) plus a background cloud.  The screened
    forward, the unscreened packet cone and the per-lane packet traversal
    must agree, no traversal stack may overflow, and sampled pixels must
    match the oracle."""
    import paper_2509_07782_b200 as G
    from paper_2509_07782_b200.scenes import synth_records

    rng = np.random.default_rng(9)
    cloud = synth_records("random-cloud", 4000, seed=3, anisotropy=2.0)
    deep = np.repeat(cloud[:1], 3200, axis=0).copy()
    deep[:3000, 0:3] = 0.05
    k = np.arange(200)
    deep[3000:, 0:3] = 0.05 + 0.5 * (0.9 ** k)[:, None] * np.array([1.0, 0.7, 0.4])
    deep[:, 7:10] = 2e-3 * rng.uniform(0.6, 1.4, (3200, 3))
    rec = f32_records(np.concatenate([cloud, deep]))
    scene = G.Scene.from_records(rec)
    G.reorder_by_morton(scene)
    cam = G.look_at_camera([0.9, 0.6, -2.2], [0.05, 0.05, 0.05], 400.0, 96, 64)
    for mode in ("adaptive", "uniform"):
        cfg = G.RenderConfig(mode=mode)
        a = G.render(scene, cam, cfg)[0].cpu().numpy()
        b = G.render(scene, cam, cfg, screen=False, traversal=1)[0].cpu().numpy()
        c = G.render(scene, cam, cfg, screen=False, traversal=2)[0].cpu().numpy()
        scene.check_render_status()
        assert np.abs(a - b).max() < 2e-6  # same arithmetic, other fp32 contraction
        assert np.abs(a - c).max() < 2e-5
        rays = O.camera_rays(cam.center, cam.quat, cam.focal, cam.width, cam.height)
        sel = np.arange(0, cam.width * cam.height, 7)
        R, T, D, _ = O.OracleScene(rec, 0.01).march_rays(rays[sel], O.OCfg.make(mode=mode),
                                                         clip=True, threads=8)
        assert np.abs(a.reshape(-1, 3)[sel] - R).max() < 1e-4
