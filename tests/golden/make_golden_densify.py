"""Golden vectors for the densification statistics, from the REFERENCE.

Run in the build container only (imports /root/reference/pkg/src):

    python tests/golden/make_golden_densify.py

The test_densify.py setup (5 random-cloud primitives, 12x12, uniform dt=0.02,
mean 0 shifted by 0.05) with a target offset by +0.03 so every residual is
non-zero and the reference's central differences are not sitting on the L1
kink; `observe_scene` (densify.py:190-204) is run for all primitives and both
loss mixes, and its accumulator arrays are stored.  Writes densify.npz.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT))

from gsray.densify import GradAccumulator, LossConfig, observe_scene  # noqa: E402
from gsray.renderer import RenderConfig, render_image  # noqa: E402
from gsray.scene_io import gen_test_scene, orbit_cameras  # noqa: E402

from make_golden import cam_arrays, ref_records, scene_from_records  # noqa: E402


def main():
    scene = scene_from_records(ref_records(gen_test_scene("random-cloud", count=5, seed=3)))
    cam = orbit_cameras(1, radius=3.0, focal=16.0, width=12, height=12)[0]
    rcfg = RenderConfig(dt=0.02)
    target, _ = render_image(scene, cam, rcfg)
    target = target + 0.03
    shifted = scene.with_mean(0, scene.means[0] + np.array([0.05, 0, 0]))
    out = {"records": ref_records(shifted), "target": target}
    out.update({f"cam.{k}": v for k, v in cam_arrays(cam).items()})
    for li, lc in ((0, LossConfig(mix=0.0)), (1, LossConfig())):
        acc = GradAccumulator(len(shifted))
        observe_scene(acc, shifted, cam, target, render_cfg=rcfg, loss_cfg=lc)
        out[f"mix{li}"] = np.array(lc.mix)
        out[f"sum_raw{li}"] = acc.sum_raw
        out[f"sum_weighted{li}"] = acc.sum_weighted
        out[f"counts{li}"] = acc.counts
    np.savez_compressed(OUT / "densify.npz", **out)
    print({k: v for k, v in out.items() if k.startswith("sum_raw")})


if __name__ == "__main__":
    main()
