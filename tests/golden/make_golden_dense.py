"""Golden vectors for the dense oracles, from the REFERENCE.

Run in the build container only (imports /root/reference/pkg/src):

    python tests/golden/make_golden_dense.py

Writes dense.npz:
* the 5-Gaussian scene of the renderer-correctness acceptance test
  (test_acceptance.py:102-133: gen_test_scene("random-cloud", 5, seed=42,
  anisotropy=2.0)) as raw records, its 24x24 reference_render at
  fine_dt = dt/8 (renderer.py:483-493) and the uniform render_image of the
  same view (renderer.py:396-437);
* reference_integrate (renderer.py:440-480) of 40 explicit rays through it,
  with a non-black background;
* eval_fields (appearance.py:107-134) at 200 points / directions, over the
  full list and over two `active` subsets.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from gsray.appearance import eval_fields  # noqa: E402
from gsray.renderer import (Ray, RenderConfig, reference_integrate, reference_render,  # noqa: E402
                            render_image)
from gsray.scene_io import gen_test_scene, orbit_cameras  # noqa: E402


def records(scene):
    rows = []
    for s, c in zip(scene.shapes, scene.coeffs):
        rows.append(np.concatenate([s.mean, s.quat, s.scales, [s.sigma], c.sh.ravel(),
                                    c.sg_axis.ravel(), c.sg_sharp.ravel(), c.sg_amp.ravel()]))
    return np.stack(rows)


def main():
    five = gen_test_scene("random-cloud", count=5, seed=42, anisotropy=2.0)
    cam = orbit_cameras(1, radius=3.0, focal=24.0, width=24, height=24)[0]
    cfg = RenderConfig()
    out = {"rec": records(five), "cam_center": cam.center, "cam_quat": cam.quat,
           "cam_focal": np.array(cam.focal), "cam_wh": np.array([cam.width, cam.height])}
    out["ref_img"] = reference_render(five, cam, cfg.dt / 8.0)
    out["march_img"] = render_image(five, cam, cfg)[0]
    rng = np.random.default_rng(5)
    rays, integ = [], []
    bg = np.array([0.2, 0.5, 0.9])
    for _ in range(40):
        o = rng.uniform(-3, 3, 3)
        d = -o + rng.normal(0, 0.3, 3)
        r = Ray(o, d, 0.5, 9.0)
        rays.append(np.concatenate([r.origin, r.direction, [r.t_near, r.t_far]]))
        integ.append(reference_integrate(five, r, 0.001, background=bg))
    out["int_rays"] = np.array(rays)
    out["int_bg"] = bg
    out["int_rgb"] = np.array(integ)
    means = np.array([s.mean for s in five.shapes])
    pts = means[rng.integers(0, 5, 200)] + rng.normal(0, 0.12, (200, 3))
    dirs = rng.normal(size=(200, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    out["f_pts"], out["f_dirs"] = pts, dirs
    for key, active in (("all", None), ("a02", [2, 0]), ("a134", [1, 3, 4])):
        fs = [eval_fields(five, x, d, active) for x, d in zip(pts, dirs)]
        out[f"f_sigma_{key}"] = np.array([f.sigma for f in fs])
        out[f"f_color_{key}"] = np.array([f.color for f in fs])
    np.savez_compressed(OUT / "dense.npz", **out)
    print("wrote", OUT / "dense.npz")


if __name__ == "__main__":
    main()
