"""Golden vectors for the render analytics (bench.py of the REFERENCE).

Run in the build container only (imports /root/reference/pkg/src):

    python tests/golden/make_golden_bench.py

Writes bench.npz: false_positive_fraction (bench.py:181-198) per ray and
overall for three anisotropy levels on 64 unclipped camera rays,
locality_metric (bench.py:236-260) for the identity and the Morton order,
and run_pipeline_matrix (bench.py:106-178) counters on a small scene.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT))

from gsray import spatial  # noqa: E402
from gsray.bench import false_positive_fraction, locality_metric, run_pipeline_matrix  # noqa
from gsray.renderer import RenderConfig  # noqa: E402
from gsray.scene_io import gen_test_scene, orbit_cameras  # noqa: E402

from make_golden import cam_arrays, ref_records, scene_from_records  # noqa: E402

LEVELS = (1.0, 4.0, 16.0)


def main():
    out = {}
    cam = orbit_cameras(1, radius=3.0, focal=12.0, width=8, height=8)[0]
    rays = [cam.ray(px, py) for py in range(8) for px in range(8)]
    out["fp.rays"] = np.array([[*r.origin, *r.direction, r.t_near, r.t_far] for r in rays])
    for li, a in enumerate(LEVELS):
        sc = scene_from_records(ref_records(gen_test_scene("random-cloud", 200, seed=4,
                                                           anisotropy=a, base_scale=0.05)))
        per_ray, overall = false_positive_fraction(sc, rays, RenderConfig())
        out[f"fp.records{li}"] = ref_records(sc)
        out[f"fp.per_ray{li}"] = per_ray
        out[f"fp.overall{li}"] = np.array(overall)
    sc = scene_from_records(ref_records(gen_test_scene("random-cloud", 500, seed=9)))
    means = sc.means
    out["loc.means"] = means
    out["loc.identity"] = np.array(locality_metric(means))
    perm = spatial.morton_order(means, sc.bounds_lo, sc.bounds_hi)
    out["loc.perm"] = perm
    out["loc.morton"] = np.array(locality_metric(means, perm))
    small = scene_from_records(ref_records(gen_test_scene("random-cloud", 30, seed=2,
                                                          base_scale=0.1)))
    cam16 = orbit_cameras(1, radius=3.0, focal=20.0, width=16, height=16)[0]
    rep = run_pipeline_matrix(small, [cam16])
    out["pm.records"] = ref_records(small)
    out.update({f"pm.cam.{k}": v for k, v in cam_arrays(cam16).items()})
    for r in rep.rows:
        key = r.pipeline.replace("+", "_")
        out[f"pm.{key}"] = np.array([r.samples_per_ray, r.aabb_hits, r.ellipsoid_hits,
                                     r.false_positive_fraction, r.psnr_vs_reference,
                                     -1.0 if r.max_abs_diff_vs_uniform is None
                                     else r.max_abs_diff_vs_uniform])
    np.savez_compressed(OUT / "bench.npz", **out)
    print({k: v for k, v in out.items() if k.startswith(("fp.overall", "loc.", "pm.u", "pm.e"))
           and v.size < 10})


if __name__ == "__main__":
    main()
