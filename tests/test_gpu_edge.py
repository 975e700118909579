"""Edge cases of the forward path vs the float64 oracle (tolerances as in
test_gpu_parity: RGB/T max abs 1e-4, depth 1e-4 * t_far)."""

import numpy as np
import pytest

import oracle as O
from paper_2509_07782_b200.scenes import f32_records, gen_test_scene_records, synth_records

pytestmark = pytest.mark.gpu


def _cmp_rays(rec, rays, cfg_kw, clip, eps=0.01):
    import paper_2509_07782_b200 as G

    s = G.Scene.from_records(rec, sigma_eps=eps)
    rgb, depth, trans, st = G.march_rays(s, rays, G.RenderConfig(**cfg_kw), clip=clip, stats=True)
    R, T, D, ost = O.OracleScene(rec, eps).march_rays(rays, O.OCfg.make(**cfg_kw), clip=clip)
    tf = np.minimum(np.abs(rays[:, 7]), 1e3)
    assert np.max(np.abs(rgb - R)) < 1e-4
    assert np.max(np.abs(trans - T)) < 1e-4
    assert np.all(np.abs(depth - D) <= 1e-4 * np.maximum(tf, 1.0))
    return st, ost


def _cmp_camera(rec, cam, cfg_kw, eps=0.01):
    import paper_2509_07782_b200 as G

    s = G.Scene.from_records(rec, sigma_eps=eps)
    rgb, depth, trans, st = G.render_full(s, cam, G.RenderConfig(**cfg_kw))
    rays = O.camera_rays(cam.center, cam.quat, cam.focal, cam.width, cam.height)
    R, T, D, _ = O.OracleScene(rec, eps).render(rays, cam.height, cam.width, O.OCfg.make(**cfg_kw))
    assert np.max(np.abs(rgb - R)) < 1e-4
    assert np.max(np.abs(trans - T)) < 1e-4
    assert np.max(np.abs(depth - D)) < 1e-4 * 10


@pytest.mark.parametrize("n_s", [1, 5, 17, 40])
@pytest.mark.parametrize("mode", ["uniform", "adaptive"])
def test_segment_sizes(n_s, mode):
    import paper_2509_07782_b200 as G

    rec = f32_records(gen_test_scene_records("random-cloud", count=150, seed=11, anisotropy=3.0))
    cam = G.orbit_cameras(1, radius=3.0, focal=18.0, width=12, height=12)[0]
    _cmp_camera(rec, cam, dict(n_s=n_s, mode=mode))


def test_odd_image_sizes_and_tiles():
    import paper_2509_07782_b200 as G

    rec = f32_records(gen_test_scene_records("random-cloud", count=300, seed=4, anisotropy=3.0,
                                             base_scale=0.05))
    for w, h in ((37, 23), (1, 1), (16, 17), (5, 40)):
        cam = G.orbit_cameras(2, radius=3.0, focal=1.2 * max(w, h), width=w, height=h)[1]
        _cmp_camera(rec, cam, dict(mode="adaptive"))


def test_rays_from_inside_and_axis_aligned(rng):
    rec = f32_records(gen_test_scene_records("random-cloud", count=200, seed=6, anisotropy=5.0,
                                             base_scale=0.1))
    rays = []
    for _ in range(200):
        o = rng.uniform(-0.9, 0.9, 3)
        d = np.zeros(3)
        k = rng.integers(0, 3)
        d[k] = rng.choice([-1.0, 1.0])
        if rng.uniform() < 0.5:
            d[(k + 1) % 3] = rng.uniform(-0.3, 0.3)
        rays.append(np.concatenate([o, d, [1e-4, rng.uniform(0.2, 3.0)]]))
    rays = np.array(rays)
    for mode in ("uniform", "adaptive"):
        for clip in (False, True):
            st, ost = _cmp_rays(rec, rays, dict(mode=mode), clip)
            # (`segments` differs by design: the reference also counts the
            # sub-collects of hit-buffer overflow splits, renderer.py:389)
            assert st.samples == ost["samples"]


def test_degenerate_and_missing_rays():
    rec = f32_records(gen_test_scene_records("single-gaussian"))
    rays = np.array([
        [0, 0, -5, 0, 0, 1, 2.0, 1.0, ],   # t_near >= t_far
        [0, 0, -5, 0, 1, 0, 1e-4, 1e6],    # misses
        [0, 0, -5, 0, 0, 1, 1e-4, 1e6],    # hits the centre
        [0, 0, 0, 1, 0, 0, 0.0, 10.0],     # starts inside
        [5, 5, 5, -1, -1, -1, 1e-4, 1e6],  # diagonal, unnormalized direction
    ], dtype=np.float64)
    for bg in ((0.0, 0.0, 0.0), (0.1, 0.2, 0.3)):
        for clip in (False, True):
            _cmp_rays(rec, rays, dict(background=bg), clip)


def test_extreme_anisotropy_and_far_background():
    """a = 1000 needles plus a far (r = 10..50) background shell."""
    import paper_2509_07782_b200 as G

    rec = synth_records("ball", 4000, seed=3, anisotropy=1000.0, shell_fraction=0.3,
                        shell_radius=(10.0, 50.0))
    cam = G.orbit_cameras(1, radius=3.5, focal=40.0, width=24, height=16)[0]
    for mode in ("uniform", "adaptive"):
        _cmp_camera(rec, cam, dict(mode=mode))


def test_tiny_dt_dense_sampling():
    import paper_2509_07782_b200 as G

    rec = f32_records(gen_test_scene_records("random-cloud", count=20, seed=1, anisotropy=2.0))
    cam = G.orbit_cameras(1, radius=3.0, focal=24.0, width=8, height=8)[0]
    _cmp_camera(rec, cam, dict(dt=0.0005, t_eps=1e-8))


def test_load_ply_scene_on_device(tmp_path):
    """PLY -> [N,87] records -> device scene (gsx_prepare validation, BVH) ->
    render, against the oracle on the same records (tests/golden/io.npz)."""
    from conftest import golden

    import oracle as O
    import paper_2509_07782_b200 as G

    g = golden("io")
    p = tmp_path / "cloud.ply"
    p.write_bytes(g["ply_binary"].tobytes())
    scene = G.load_ply_scene(p)
    assert scene.n == 300
    np.testing.assert_array_equal(scene.records().astype(np.float32), g["records_binary"])
    cam = G.orbit_cameras(1, radius=6.0, focal=24.0, width=16, height=16)[0]
    cfg = G.RenderConfig(mode="adaptive")
    rgb = G.render(scene, cam, cfg)[0].cpu().numpy()
    osc = O.OracleScene(g["records_binary"].astype(np.float64))
    R = osc.render(O.camera_rays(cam.center, cam.quat, cam.focal, 16, 16), 16, 16,
                   O.OCfg.make(mode="adaptive"))[0]
    assert np.abs(rgb - R.reshape(16, 16, 3)).max() < 1e-4
