"""Render analytics (paper_2509_07782_b200/analysis.py) against the
reference's bench.py on tests/golden/bench.npz
(tests/golden/make_golden_bench.py): per-ray false-positive fractions and
the pipeline-matrix counters are exact (they are reference-semantics
counts); node visits are tree-dependent and PSNR uses our dense reference,
so those are only sanity-checked."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("li", [0, 1, 2])
def test_false_positive_fraction_exact(li):
    import paper_2509_07782_b200 as G
    from paper_2509_07782_b200.analysis import false_positive_fraction

    g = golden("bench")
    scene = G.Scene.from_records(g[f"fp.records{li}"].astype(np.float32))
    per_ray, overall = false_positive_fraction(scene, g["fp.rays"], G.RenderConfig())
    np.testing.assert_array_equal(per_ray, g[f"fp.per_ray{li}"])
    assert overall == float(g[f"fp.overall{li}"])


def test_isotropy_sweep_monotone():
    import paper_2509_07782_b200 as G
    from paper_2509_07782_b200.analysis import isotropy_sweep

    g = golden("bench")
    res = isotropy_sweep([0, 1, 2], lambda s: g["fp.rays"],
                         lambda li: G.Scene.from_records(g[f"fp.records{li}"].astype(np.float32)))
    for li, r in enumerate(res):
        assert r["fraction"] == float(g[f"fp.overall{li}"])
        assert r["ci_lo"] <= r["fraction"] <= r["ci_hi"]


def test_pipeline_matrix_counters():
    import paper_2509_07782_b200 as G
    from paper_2509_07782_b200.analysis import run_pipeline_matrix

    g = golden("bench")
    scene = G.Scene.from_records(g["pm.records"].astype(np.float32))
    cam = G.Camera(center=g["pm.cam.cam_center"], quat=g["pm.cam.cam_quat"],
                   focal=float(g["pm.cam.cam_focal"]), width=int(g["pm.cam.cam_w"]),
                   height=int(g["pm.cam.cam_h"]))
    rep = run_pipeline_matrix(scene, [cam], repeats=2)
    assert [r.pipeline for r in rep.rows] == ["uniform", "ess", "ess+adaptive"]
    for r in rep.rows:
        ref = g["pm." + r.pipeline.replace("+", "_")]
        assert r.samples_per_ray == pytest.approx(float(ref[0]), rel=1e-12)
        assert r.aabb_hits == int(ref[1]) and r.ellipsoid_hits == int(ref[2])
        assert r.false_positive_fraction == pytest.approx(float(ref[3]), rel=1e-12)
        assert r.psnr_vs_reference > 60.0 and r.wall_time_s > 0.0
    assert rep.rows[1].max_abs_diff_vs_uniform <= 1e-6  # ESS is lossless (reference: 0.0)
    assert rep.to_csv().splitlines()[0].startswith("pipeline,samples_per_ray")
