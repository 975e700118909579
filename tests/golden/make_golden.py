"""Generate golden vectors by running the REFERENCE (`gsray`, pure Python).

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Every scene is first rounded to float32 records
(the .gsx wire format, scene_io.py:44) and re-ingested the way
`scene_io.load_scene` does (scene_io.py:84-105), so the reference, the oracle
and the GPU all consume identical parameters.
"""

from __future__ import annotations

import hashlib
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(OUT.parent.parent))

from gsray import spatial  # noqa: E402
from gsray.appearance import AppearanceCoeffs, eval_radiance  # noqa: E402
from gsray.densify import LossConfig, _ssim, fd_position_gradient, image_loss  # noqa: E402
from gsray.geometry import GaussianShape  # noqa: E402
from gsray.renderer import (Camera, RenderConfig, RenderStats, clip_ray_to_scene,  # noqa: E402
                            march_ray, render_image, segment_step)
from gsray.scene import Scene, reorder_by_morton  # noqa: E402
from gsray.scene_io import _record, gen_test_scene, orbit_cameras  # noqa: E402

from paper_2509_07782_b200.scenes import gen_test_scene_records  # noqa: E402


def ref_records(scene) -> np.ndarray:
    return np.stack([_record(s, c) for s, c in zip(scene.shapes, scene.coeffs)]).astype(
        np.float64)


def scene_from_records(rec: np.ndarray, sigma_eps: float = 0.01) -> Scene:
    """scene_io.py:84-105 without the file."""
    shapes, coeffs = [], []
    for r in rec:
        shapes.append(GaussianShape(mean=r[0:3], quat=r[3:7], scales=r[7:10], sigma=float(r[10])))
        coeffs.append(AppearanceCoeffs(r[11:38].reshape(9, 3), r[38:59].reshape(7, 3),
                                       r[59:66], r[66:87].reshape(7, 3)))
    return Scene(shapes, coeffs, sigma_eps=sigma_eps)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# -- per-pixel march over a camera (fork pool, rows interleaved) -------------
_G = {}


def _row(py):
    scene, cam, cfg = _G["scene"], _G["cam"], _G["cfg"]
    px_list = _G["px"]
    out = []
    for px in px_list:
        ray0 = cam.ray(px, py)
        ray = clip_ray_to_scene(scene, ray0)
        st = RenderStats()
        if ray is None:
            out.append((px, py, list(cfg.background), 1.0, [np.nan] * 8, None))
            continue
        rgb, st = march_ray(scene, ray, cfg, stats=st)
        rv = list(ray.origin) + list(ray.direction) + [ray.t_near, ray.t_far]
        out.append((px, py, list(rgb), st.transmittance, rv,
                    [st.samples, st.segments, st.segments_skipped, st.closest_hit_calls,
                     st.aabb_hits, st.ellipsoid_hits]))
    return out


def render_pixels(scene, cam, cfg, rows=None, cols=None, procs=8):
    rows = list(range(cam.height)) if rows is None else list(rows)
    cols = list(range(cam.width)) if cols is None else list(cols)
    _G.update(scene=scene, cam=cam, cfg=cfg, px=cols)
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        res = pool.map(_row, rows, chunksize=1)
    H, W = len(rows), len(cols)
    rgb = np.zeros((H, W, 3))
    T = np.zeros((H, W))
    rays = np.full((H, W, 8), np.nan)
    st = np.zeros(6, dtype=np.int64)
    for ri, row in enumerate(res):
        for ci, (px, py, c, t, rv, s) in enumerate(row):
            rgb[ri, ci] = c
            T[ri, ci] = t
            rays[ri, ci] = rv
            if s is not None:
                st += np.array(s, dtype=np.int64)
    return rgb, T, rays, st


def cam_arrays(cam: Camera):
    return dict(cam_center=np.asarray(cam.center), cam_quat=np.asarray(cam.quat),
                cam_focal=float(cam.focal), cam_w=cam.width, cam_h=cam.height)


CFGS = {
    "uniform": RenderConfig(),
    "uniform_noess": RenderConfig(ess=False),
    "adaptive": RenderConfig(mode="adaptive"),
    "adaptive_noess": RenderConfig(mode="adaptive", ess=False),
    "uniform_bg_cap2": RenderConfig(background=(0.1, 0.2, 0.3), buffer_capacity=2),
}


def main():
    t_start = time.time()
    # ---------------------------------------------------------------- scenes
    specs = {
        "small": dict(kind="random-cloud", count=20, seed=1),
        "grid": dict(kind="grid", count=27, seed=3),
        "shell": dict(kind="shell", count=12, seed=5),
        "single": dict(kind="single-gaussian"),
        "q150": dict(kind="random-cloud", count=150, seed=11, anisotropy=3.0),
        "q100": dict(kind="random-cloud", count=100, seed=7, anisotropy=3.0),
        "q30": dict(kind="random-cloud", count=30, seed=17, anisotropy=3.0),
        "c1": dict(kind="random-cloud", count=10_000, seed=0, anisotropy=3.0,
                   base_scale=0.01177),
    }
    gen = {}
    ref_scenes = {}
    for name, sp in specs.items():
        ref = gen_test_scene(**sp)
        r64 = ref_records(ref)                       # reference, float32 -> f64 via _record
        mine = gen_test_scene_records(**sp)          # our generator, float64
        mine32 = mine.astype(np.float32).astype(np.float64)
        assert np.array_equal(mine32, r64), f"generator mismatch for {name}"
        # exact float64 equality of the generator before f32 rounding
        full = np.stack([np.concatenate([s.mean, s.quat, s.scales, [s.sigma], c.sh.ravel(),
                                         c.sg_axis.ravel(), c.sg_sharp, c.sg_amp.ravel()])
                         for s, c in zip(ref.shapes, ref.coeffs)])
        gen[name] = dict(sha_f64=sha(full), sha_f32=sha(r64), exact_f64=bool(np.array_equal(full, mine)))
        ref_scenes[name] = scene_from_records(r64)
        print(name, "generator f64 exact:", gen[name]["exact_f64"], flush=True)

    np.savez_compressed(OUT / "generator.npz",
                        names=np.array(list(gen)),
                        sha_f64=np.array([gen[k]["sha_f64"] for k in gen]),
                        sha_f32=np.array([gen[k]["sha_f32"] for k in gen]),
                        exact_f64=np.array([gen[k]["exact_f64"] for k in gen]))

    # -------------------------------------------------------- derived arrays
    d = {}
    for name in ("small", "grid", "shell", "single", "q150"):
        s = ref_scenes[name]
        for attr in ("means", "rotations", "scales", "sigmas", "log_ratio", "iso_scales",
                     "iso_inv", "aabb_lo", "aabb_hi", "bounds_lo", "bounds_hi"):
            d[f"{name}.{attr}"] = np.asarray(getattr(s, attr))
    s = ref_scenes["c1"]
    d["c1.bounds_lo"] = s.bounds_lo
    d["c1.bounds_hi"] = s.bounds_hi
    d["c1.aabb_lo"] = s.aabb_lo.astype(np.float64)
    d["c1.aabb_hi"] = s.aabb_hi.astype(np.float64)
    np.savez_compressed(OUT / "derived.npz", **d)

    # ------------------------------------------------------------- morton
    m = {}
    rng = np.random.default_rng(1234)
    pts = rng.integers(0, spatial.MORTON_MAX + 1, size=(100, 3))
    m["enc_pts"] = pts
    m["enc_codes"] = spatial.morton_encode(pts).astype(np.uint64)
    s = ref_scenes["c1"]
    q = spatial.quantize_points(s.means, s.bounds_lo, s.bounds_hi)
    m["c1.quant"] = q
    m["c1.codes"] = spatial.morton_encode(q).astype(np.uint64)
    m["c1.perm"] = spatial.morton_order(s.means, s.bounds_lo, s.bounds_hi)
    for name in ("small", "grid", "shell", "q150"):
        sc = scene_from_records(ref_records(gen_test_scene(**specs[name])))
        m[f"{name}.perm"] = reorder_by_morton(sc)
        m[f"{name}.perm2"] = reorder_by_morton(sc)  # idempotent: identity
        m[f"{name}.uids_after"] = sc.uids.copy()
    # duplicate-heavy codes: stability of the sort
    dup = np.repeat(rng.uniform(-1, 1, size=(50, 3)), 7, axis=0)
    rng.shuffle(dup)
    m["dup.pts"] = dup
    m["dup.perm"] = spatial.morton_order(dup, dup.min(0), dup.max(0))
    np.savez_compressed(OUT / "morton.npz", **m)
    print("morton done", flush=True)

    # ------------------------------------------------------------- queries
    qd = {}
    rng = np.random.default_rng(1234)
    s = ref_scenes["q150"]
    buf = spatial.HitBuffer(capacity=256)
    Q, sets, offs = [], [], [0]
    for _ in range(300):
        o = rng.uniform(-2, 2, 3)
        dd = rng.standard_normal(3)
        dd /= np.linalg.norm(dd)
        t0 = rng.uniform(0, 3)
        t1 = t0 + rng.uniform(0, 2)
        s.bvh.segment_overlaps(o, dd, t0, t1, buf)
        got = sorted(buf.active().tolist())
        Q.append(np.concatenate([o, dd, [t0, t1]]))
        sets.extend(got)
        offs.append(len(sets))
    # axis-aligned and zero-component directions, degenerate segments
    for _ in range(100):
        o = rng.uniform(-1.2, 1.2, 3)
        dd = np.zeros(3)
        ax = rng.integers(0, 3)
        dd[ax] = rng.choice([-1.0, 1.0])
        t0 = rng.uniform(0, 1)
        t1 = t0 + rng.choice([0.0, rng.uniform(0, 1)])
        s.bvh.segment_overlaps(o, dd, t0, t1, buf)
        got = sorted(buf.active().tolist())
        Q.append(np.concatenate([o, dd, [t0, t1]]))
        sets.extend(got)
        offs.append(len(sets))
    qd["q150.queries"] = np.array(Q)
    qd["q150.sets"] = np.array(sets, dtype=np.int64)
    qd["q150.offsets"] = np.array(offs, dtype=np.int64)
    for name, nq, seed in (("q100", 300, 7), ("q30", 2000, 31)):
        s = ref_scenes[name]
        rng = np.random.default_rng(seed)
        Q, H = [], []
        for _ in range(nq):
            o = rng.uniform(-2, 2, 3)
            dd = rng.standard_normal(3)
            dd /= np.linalg.norm(dd)
            t0 = rng.uniform(0, 2)
            t1 = t0 + rng.uniform(0, 3)
            h = spatial.closest_hit(s.bvh, s, o, dd, t0, t1)
            Q.append(np.concatenate([o, dd, [t0, t1]]))
            H.append(np.nan if h is None else h)
        qd[f"{name}.queries"] = np.array(Q)
        qd[f"{name}.hits"] = np.array(H)
    np.savez_compressed(OUT / "queries.npz", **qd)
    print("queries done", flush=True)

    # --------------------------------------------------------- small renders
    rd = {}
    cam16 = orbit_cameras(1, radius=3.0, focal=24.0, width=16, height=16)[0]
    rd.update({f"cam16.{k}": v for k, v in cam_arrays(cam16).items()})
    for sname in ("small", "grid", "shell", "single"):
        s = ref_scenes[sname]
        cfg_names = CFGS if sname == "small" else {"uniform": CFGS["uniform"],
                                                    "adaptive": CFGS["adaptive"]}
        for cname in cfg_names:
            cfg = CFGS[cname]
            rgb, T, rays, st = render_pixels(s, cam16, cfg)
            img, stats = render_image(s, cam16, cfg)
            assert np.array_equal(img, rgb)
            rd[f"{sname}.{cname}.rgb"] = rgb
            rd[f"{sname}.{cname}.T"] = T
            rd[f"{sname}.{cname}.rays"] = rays
            rd[f"{sname}.{cname}.stats"] = np.array(
                [stats.rays, stats.samples, stats.segments, stats.segments_skipped,
                 stats.closest_hit_calls, stats.node_visits, stats.aabb_hits,
                 stats.ellipsoid_hits], dtype=np.int64)
    # a second camera pose, wider fov, non-square
    cam_b = orbit_cameras(3, radius=2.5, focal=14.0, width=20, height=12)[1]
    rd.update({f"camb.{k}": v for k, v in cam_arrays(cam_b).items()})
    for cname in ("uniform", "adaptive"):
        rgb, T, rays, st = render_pixels(ref_scenes["q150"], cam_b, CFGS[cname])
        rd[f"q150.{cname}.rgb"] = rgb
        rd[f"q150.{cname}.T"] = T
    np.savez_compressed(OUT / "render_small.npz", **rd)
    print("small renders done", time.time() - t_start, flush=True)

    # ------------------------------------------------------------ C1 render
    c1 = {}
    cam64 = orbit_cameras(1, radius=3.0, focal=64.0, width=64, height=64)[0]
    c1.update({f"cam64.{k}": v for k, v in cam_arrays(cam64).items()})
    t0 = time.time()
    rgb, T, rays, st = render_pixels(ref_scenes["c1"], cam64, CFGS["uniform"])
    c1["c1.uniform.rgb"] = rgb
    c1["c1.uniform.T"] = T
    c1["c1.uniform.rays"] = rays
    c1["c1.uniform.stats6"] = st
    c1["c1.uniform.seconds_8proc"] = time.time() - t0
    print("c1 uniform", time.time() - t0, flush=True)
    sub = list(range(0, 64, 4))
    rgb, T, rays, st = render_pixels(ref_scenes["c1"], cam64, CFGS["adaptive"], rows=sub, cols=sub)
    c1["c1.adaptive_sub4.rgb"] = rgb
    c1["c1.adaptive_sub4.T"] = T
    np.savez_compressed(OUT / "render_c1.npz", **c1)
    print("c1 done", flush=True)

    # -------------------------------------------------------- misc numerics
    mi = {}
    cfg = RenderConfig(mode="adaptive")
    rng = np.random.default_rng(5)
    dv = rng.uniform(0.0, 200.0, 300)
    tv = np.concatenate([rng.uniform(0, 1, 290), [0.0, 1e-5, 1e-4, 1.0, 0.5, 1e-30, 0.125,
                                                 0.3, 0.9, 0.999]])
    mi["step.d"] = dv
    mi["step.t"] = tv
    mi["step.val"] = np.array([segment_step(cfg, a, b) for a, b in zip(dv, tv)])
    s = ref_scenes["small"]
    dirs = rng.standard_normal((50, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    mi["rad.dirs"] = dirs
    mi["rad.val"] = np.array([[eval_radiance(s.coeffs[i], dd) for dd in dirs]
                              for i in range(len(s))])
    # loss
    rng = np.random.default_rng(1234)
    a = rng.uniform(size=(32, 32, 3))
    b = np.clip(a + rng.normal(0, 0.1, a.shape), 0, 1)
    mi["loss.a"] = a
    mi["loss.b"] = b
    mi["loss.ssim"] = _ssim(a, b)
    mi["loss.total"] = image_loss(a, b, LossConfig())
    g1 = rng.uniform(size=(40, 36))
    g2 = np.clip(g1 + rng.normal(0, 0.1, g1.shape), 0, 1)
    mi["loss.g1"] = g1
    mi["loss.g2"] = g2
    mi["loss.ssim_gray"] = _ssim(g1, g2)
    # reference FD position gradient (densify.py:156-187), test_densify setup
    scene = scene_from_records(ref_records(gen_test_scene("random-cloud", count=5, seed=3)))
    cam12 = orbit_cameras(1, radius=3.0, focal=16.0, width=12, height=12)[0]
    rcfg = RenderConfig(dt=0.02)
    target, _ = render_image(scene, cam12, rcfg)
    shifted = scene.with_mean(0, scene.means[0] + np.array([0.05, 0, 0]))
    mi["fd.records"] = ref_records(scene)
    mi["fd.target"] = target
    mi["fd.shift"] = np.array([0.05, 0, 0])
    mi.update({f"cam12.{k}": v for k, v in cam_arrays(cam12).items()})
    for li, lc in ((0, LossConfig(mix=0.0)), (1, LossConfig())):
        mi[f"fd.grad{li}"] = np.stack([fd_position_gradient(shifted, cam12, target, i,
                                                            render_cfg=rcfg, loss_cfg=lc)
                                       for i in range(5)])
    np.savez_compressed(OUT / "misc.npz", **mi)
    print("all done", time.time() - t_start, flush=True)


if __name__ == "__main__":
    main()
