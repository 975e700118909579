"""The packet-cone paths of the camera kernel (cone traversal, cone-window ESS
closest hit; render.cu / render_warp.cuh) against the per-lane packet paths
of the explicit-ray kernel on the very same rays, and against the oracle,
over the cameras the cone construction has to survive: wide fields of view,
cameras inside the scene, off-image lanes (tiles cut by the image border),
lanes whose rays miss the scene, and a large far background."""

import numpy as np
import pytest

import oracle as O
from paper_2509_07782_b200.scenes import f32_records, gen_test_scene_records, synth_records

pytestmark = pytest.mark.gpu


def _both(G, scene, cam, cfg):
    rgb, depth, trans, st = G.render_full(scene, cam, cfg)
    rays = O.camera_rays(cam.center, cam.quat, cam.focal, cam.width, cam.height)
    r2, d2, t2, st2 = G.march_rays(scene, rays, cfg, clip=True, stats=True)
    h, w = cam.height, cam.width
    return (rgb, depth, trans, st), (r2.reshape(h, w, 3), d2.reshape(h, w), t2.reshape(h, w), st2)


CAMS = [  # (radius, focal, width, height): narrow, wide, very wide, odd tiles
    (3.0, 64.0, 48, 40), (3.0, 10.0, 20, 12), (2.0, 4.0, 33, 17), (0.3, 12.0, 24, 24),
]


@pytest.mark.parametrize("mode", ["uniform", "adaptive"])
@pytest.mark.parametrize("cam_i", range(len(CAMS)))
def test_cone_paths_match_per_lane_paths(mode, cam_i):
    """Camera kernel (cone traversal + cone ESS) == explicit-ray kernel (per-lane
    packet traversal + packet ESS) on the same rays: the candidate lists differ
    (superset, other order), so sums agree to fp32 rounding; every RenderStats
    counter except node visits is identical (same ESS jumps, same segments)."""
    import paper_2509_07782_b200 as G

    rec = f32_records(gen_test_scene_records("random-cloud", count=400, seed=21, anisotropy=3.0,
                                             base_scale=0.06))
    scene = G.Scene.from_records(rec)
    G.reorder_by_morton(scene)
    radius, focal, w, h = CAMS[cam_i]
    cam = G.orbit_cameras(3, radius=radius, focal=focal, width=w, height=h)[cam_i % 3]
    cfg = G.RenderConfig(mode=mode)
    (rgb, depth, trans, st), (r2, d2, t2, st2) = _both(G, scene, cam, cfg)
    assert np.max(np.abs(rgb - r2)) < 2e-5
    assert np.max(np.abs(trans - t2)) < 2e-5
    assert np.max(np.abs(depth - d2)) < 1e-4
    for k in ("rays", "samples", "segments", "segments_skipped", "closest_hit_calls",
              "aabb_hits", "ellipsoid_hits"):
        assert getattr(st, k) == getattr(st2, k), k


def test_cone_far_background_vs_oracle():
    """C3-shaped scene (dense ball + far background shell, scale ~ distance):
    ESS windows have to double across the empty gap to the shell."""
    import paper_2509_07782_b200 as G

    rec = synth_records("ball", 3000, seed=2, anisotropy=3.0, r_max_bound=10.0,
                        shell_fraction=0.3, shell_radius=(10.0, 50.0))
    scene = G.Scene.from_records(rec)
    G.reorder_by_morton(scene)
    cam = G.orbit_cameras(1, radius=3.5, focal=1.2 * 40, width=40, height=24)[0]
    for mode in ("adaptive", "uniform"):
        cfg = G.RenderConfig(mode=mode)
        rgb, depth, trans, _ = G.render_full(scene, cam, cfg)
        rays = O.camera_rays(cam.center, cam.quat, cam.focal, cam.width, cam.height)
        R, T, D, _ = O.OracleScene(rec, 0.01).render(rays, cam.height, cam.width,
                                                      O.OCfg.make(mode=mode))
        assert np.max(np.abs(rgb - R)) < 1e-4
        assert np.max(np.abs(trans - T)) < 1e-4


@pytest.mark.parametrize("min_focal", ["0", "1e30"])
def test_plain_forward_traversal_choice(monkeypatch, min_focal):
    """The plain whole-image / sharded forward picks the packet cone for
    focal >= GSX_CONE_MIN_FOCAL and the per-lane packet traversal below it;
    both equal the oracle (forced here through the environment override)."""
    import torch

    import paper_2509_07782_b200 as G

    monkeypatch.setenv("GSX_CONE_MIN_FOCAL", min_focal)
    rec = synth_records("ball", 3000, seed=2, anisotropy=3.0, r_max_bound=10.0,
                        shell_fraction=0.3, shell_radius=(10.0, 50.0))
    scene = G.Scene.from_records(rec)
    G.reorder_by_morton(scene)
    cam = G.orbit_cameras(1, radius=3.5, focal=1.2 * 40, width=40, height=24)[0]
    cfg = G.RenderConfig(mode="adaptive")
    rays = O.camera_rays(cam.center, cam.quat, cam.focal, cam.width, cam.height)
    R, T, D, _ = O.OracleScene(rec, 0.01).render(rays, cam.height, cam.width,
                                                  O.OCfg.make(mode="adaptive"))
    rgb, depth, trans, _ = G.render(scene, cam, cfg)
    assert np.max(np.abs(rgb.cpu().numpy() - R)) < 1e-4
    assert np.max(np.abs(trans.cpu().numpy() - T)) < 1e-4
    out = torch.zeros_like(rgb)
    for r in range(2):
        G.render(scene, cam, cfg, tile_begin=r, tile_stride=2, rgb=out)
    assert np.max(np.abs(out.cpu().numpy() - R)) < 1e-4
