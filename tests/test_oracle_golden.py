"""Pin the CPU oracle (oracle/gsray_oracle.c) against golden vectors produced
by the reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle as O
from conftest import golden
from paper_2509_07782_b200.scenes import f32_records, gen_test_scene_records

SPECS = {
    "small": dict(kind="random-cloud", count=20, seed=1),
    "grid": dict(kind="grid", count=27, seed=3),
    "shell": dict(kind="shell", count=12, seed=5),
    "single": dict(kind="single-gaussian"),
    "q150": dict(kind="random-cloud", count=150, seed=11, anisotropy=3.0),
    "q100": dict(kind="random-cloud", count=100, seed=7, anisotropy=3.0),
    "q30": dict(kind="random-cloud", count=30, seed=17, anisotropy=3.0),
    "c1": dict(kind="random-cloud", count=10_000, seed=0, anisotropy=3.0, base_scale=0.01177),
}

_cache = {}


def oscene(name):
    if name not in _cache:
        _cache[name] = O.OracleScene(f32_records(gen_test_scene_records(**SPECS[name])))
    return _cache[name]


def test_generator_matches_reference():
    import hashlib

    g = golden("generator")
    for name, want, exact in zip(g["names"], g["sha_f32"], g["exact_f64"]):
        rec = f32_records(gen_test_scene_records(**SPECS[str(name)]))
        assert hashlib.sha256(rec.tobytes()).hexdigest() == want, name
        assert bool(exact)


@pytest.mark.parametrize("name", ["small", "grid", "shell", "single", "q150"])
def test_derived_arrays(name):
    g = golden("derived")
    s = oscene(name)
    for attr in ("means", "scales", "sigmas", "log_ratio"):
        assert np.array_equal(s.get(attr), g[f"{name}.{attr}"]), attr
    for attr in ("rotations", "iso_scales", "iso_inv", "aabb_lo", "aabb_hi"):
        np.testing.assert_allclose(s.get(attr), g[f"{name}.{attr}"], rtol=0, atol=1e-13)
    lo, hi = s.get("bounds")
    np.testing.assert_allclose(lo, g[f"{name}.bounds_lo"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(hi, g[f"{name}.bounds_hi"], rtol=0, atol=1e-15)


def test_c1_bounds_bit_exact():
    g = golden("derived")
    lo, hi = oscene("c1").get("bounds")
    assert np.array_equal(lo, g["c1.bounds_lo"]) and np.array_equal(hi, g["c1.bounds_hi"])


class TestMorton:
    def test_known_answers(self):
        # test_spatial.py:24-33
        assert O.morton_encode([0, 0, 0])[0] == 0
        assert O.morton_encode([1, 1, 1])[0] == 7
        assert O.morton_encode([3, 1, 0])[0] == 11
        assert list(O.morton_decode(11)[0]) == [3, 1, 0]

    def test_boundary_roundtrip(self):
        mx = (1 << 21) - 1
        for v in (0, 1, mx - 1, mx):
            p = [v, mx - v, v // 2]
            assert list(O.morton_decode(O.morton_encode(p))[0]) == p

    def test_out_of_range(self):
        with pytest.raises(ValueError):
            O.morton_encode([1 << 21, 0, 0])

    def test_encode_golden(self):
        g = golden("morton")
        assert np.array_equal(O.morton_encode(g["enc_pts"]), g["enc_codes"])

    def test_c1_codes_and_perm_bit_exact(self):
        g = golden("morton")
        s = oscene("c1")
        lo, hi = s.get("bounds")
        assert np.array_equal(O.quantize_points(s.get("means"), lo, hi), g["c1.quant"])
        codes, perm = O.morton_order(s.get("means"), lo, hi)
        assert np.array_equal(codes, g["c1.codes"])
        assert np.array_equal(perm, g["c1.perm"])

    @pytest.mark.parametrize("name", ["small", "grid", "shell", "q150"])
    def test_reorder(self, name):
        g = golden("morton")
        s = O.OracleScene(f32_records(gen_test_scene_records(**SPECS[name])))
        assert np.array_equal(s.reorder_by_morton(), g[f"{name}.perm"])
        assert np.array_equal(s.reorder_by_morton(), g[f"{name}.perm2"])
        assert np.array_equal(s.get("uids"), g[f"{name}.uids_after"])

    def test_stability_with_duplicates(self):
        g = golden("morton")
        pts = g["dup.pts"]
        _, perm = O.morton_order(pts, pts.min(0), pts.max(0))
        assert np.array_equal(perm, g["dup.perm"])


class TestQueries:
    def test_segment_sets_bit_exact(self):
        g = golden("queries")
        s = oscene("q150")
        Q, offs, sets = g["q150.queries"], g["q150.offsets"], g["q150.sets"]
        for i, q in enumerate(Q):
            want = sets[offs[i]:offs[i + 1]]
            assert np.array_equal(s.segment_overlaps(q[:3], q[3:6], q[6], q[7]), want)
            assert np.array_equal(s.segment_overlaps_brute(q[:3], q[3:6], q[6], q[7]), want)

    @pytest.mark.parametrize("name", ["q100", "q30"])
    def test_closest_hit(self, name):
        g = golden("queries")
        s = oscene(name)
        for q, h in zip(g[f"{name}.queries"], g[f"{name}.hits"]):
            t = s.closest_hit(q[:3], q[3:6], q[6], q[7])
            if np.isnan(h):
                assert t is None
            else:
                assert t is not None and abs(t - h) < 1e-9

    def test_overflow(self):
        s = oscene("q150")
        with pytest.raises(O.OracleError):
            s.segment_overlaps([-3.0, 0, 0], [1.0, 0, 0], 0.0, 8.0, capacity=1)

    def test_grazing(self):
        # test_spatial.py:238-249
        hit = O.ray_ellipsoid_interval([-10.0, 1.0 - 1e-9, 0.0], [1.0, 0, 0], 0.0, 100.0)
        assert hit is not None and abs(hit[0] - 10.0) < 1e-2
        assert O.ray_ellipsoid_interval([-10.0, 2.0, 0.0], [1.0, 0, 0], 0.0, 100.0) is None


CFG = {
    "uniform": {}, "uniform_noess": dict(ess=False), "adaptive": dict(mode="adaptive"),
    "adaptive_noess": dict(mode="adaptive", ess=False),
    "uniform_bg_cap2": dict(background=(0.1, 0.2, 0.3), buffer_capacity=2),
}


def cam_rays(g, prefix):
    return O.camera_rays(g[f"{prefix}.cam_center"], g[f"{prefix}.cam_quat"],
                         float(g[f"{prefix}.cam_focal"]), int(g[f"{prefix}.cam_w"]),
                         int(g[f"{prefix}.cam_h"]))


@pytest.mark.parametrize("scene,cname", [("small", c) for c in CFG] +
                         [(s, c) for s in ("grid", "shell", "single") for c in ("uniform", "adaptive")])
def test_render_small(scene, cname):
    g = golden("render_small")
    rays = cam_rays(g, "cam16")
    rgb, T, D, st = oscene(scene).render(rays, 16, 16, O.OCfg.make(**CFG[cname]))
    np.testing.assert_allclose(rgb, g[f"{scene}.{cname}.rgb"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(T, g[f"{scene}.{cname}.T"], rtol=0, atol=1e-12)
    ref = g[f"{scene}.{cname}.stats"]
    got = [st[k] for k in ("rays", "samples", "segments", "segments_skipped",
                           "closest_hit_calls")]
    assert got == list(ref[:5])
    assert st["aabb_hits"] == ref[6] and st["ellipsoid_hits"] == ref[7]


def test_render_camera_b():
    g = golden("render_small")
    rays = cam_rays(g, "camb")
    for cname in ("uniform", "adaptive"):
        rgb, T, D, st = oscene("q150").render(rays, 12, 20, O.OCfg.make(**CFG[cname]))
        np.testing.assert_allclose(rgb, g[f"q150.{cname}.rgb"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(T, g[f"q150.{cname}.T"], rtol=0, atol=1e-12)


def test_clipped_rays_match():
    g = golden("render_small")
    rays = cam_rays(g, "cam16")
    want = g["small.uniform.rays"].reshape(-1, 8)
    np.testing.assert_allclose(rays[:, :6], np.where(np.isnan(want[:, :6]), rays[:, :6],
                                                     want[:, :6]), atol=1e-15)


def test_render_c1_full_frame():
    g = golden("render_c1")
    rays = cam_rays(g, "cam64")
    rgb, T, D, st = oscene("c1").render(rays, 64, 64, O.OCfg.make(), threads=4)
    np.testing.assert_allclose(rgb, g["c1.uniform.rgb"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(T, g["c1.uniform.T"], rtol=0, atol=1e-12)
    ref = g["c1.uniform.stats6"]
    assert [st["samples"], st["segments"], st["segments_skipped"], st["closest_hit_calls"],
            st["aabb_hits"], st["ellipsoid_hits"]] == list(ref)


def test_render_c1_adaptive_subset():
    g = golden("render_c1")
    rays = cam_rays(g, "cam64").reshape(64, 64, 8)[::4, ::4].reshape(-1, 8)
    rgb, T, D, st = oscene("c1").march_rays(rays, O.OCfg.make(mode="adaptive"), threads=4)
    np.testing.assert_allclose(rgb.reshape(16, 16, 3), g["c1.adaptive_sub4.rgb"], atol=1e-12)
    np.testing.assert_allclose(T.reshape(16, 16), g["c1.adaptive_sub4.T"], atol=1e-12)


def test_segment_step_and_radiance():
    g = golden("misc")
    cfg = O.OCfg.make(mode="adaptive")
    got = np.array([O.segment_step(cfg, a, b) for a, b in zip(g["step.d"], g["step.t"])])
    np.testing.assert_allclose(got, g["step.val"], rtol=1e-15, atol=0)
    assert abs(O.segment_step(O.OCfg.make(mode="adaptive"), 10.24, 0.125) - 0.32) < 1e-12
    s = oscene("small")
    for i in range(len(s)):
        for dv, want in zip(g["rad.dirs"], g["rad.val"][i]):
            np.testing.assert_allclose(s.eval_radiance(i, dv), want, rtol=0, atol=1e-14)
