"""B200-native RayGaussX volumetric ray marcher: a drop-in for the render path
of the reference package `gsray` (/root/reference/pkg/src/gsray/__init__.py).

Same entry-point names and layouts; the work runs in hand-written sm_100a
kernels (libgsx.so, C ABI in include/gsx.h).  There is no CPU fallback.
"""

from .appearance import (AppearanceCoeffs, FieldSample, eval_fields, eval_fields_batch,
                         eval_radiance, sh_basis)
from .config import Camera, Ray, RenderConfig, RenderStats, quat_to_rotation, segment_step
from .geometry import (Aabb, GaussianShape, IsoLossConfig, aabb_of, ellipsoid_volume, iso_scale,
                       isotropic_loss, ratio_upper_bound, volume_ratio)
from .densify import (DensifyConfig, GradAccumulator, criterion_new, criterion_old,
                      fd_position_gradient, neighbor_density, observe_scene)
from .errors import (BufferOverflow, DegenerateCenter, EmptyIsosurface, EmptyScene, GsrayError,
                     ParseError, TraversalOverflow, ValidationError)
from .renderer import (VARIANTS, MarchLog, autotune, clip_ray_to_scene, march_ray, march_rays,
                       psnr, reference_integrate, reference_render, reference_rays, render,
                       render_backward, render_full, render_image)
from .scene import Scene, gen_test_scene, load_scene, reorder_by_morton, save_scene
from .scene_io import (load_cameras, load_ply_scene, ply_records,
                       save_cameras)
from .scenes import orbit_poses, look_at


def orbit_cameras(n, radius, focal, width, height, elevation=0.35, target=(0.0, 0.0, 0.0)):
    """scene_io.py:175-187."""
    return [Camera(center=c, quat=q, focal=focal, width=width, height=height)
            for c, q in orbit_poses(n, radius, elevation, target)]


def look_at_camera(center, target, focal, width, height, up=(0.0, 1.0, 0.0), **kw):
    """scene_io.py:158-172."""
    c, q = look_at(center, target, up)
    return Camera(center=c, quat=q, focal=focal, width=width, height=height, **kw)


__all__ = [
    # the reference's public names (gsray/__init__.py:6-52)
    "Aabb", "AppearanceCoeffs", "BufferOverflow", "Camera", "DegenerateCenter",
    "EmptyIsosurface", "EmptyScene", "FieldSample", "GaussianShape", "GsrayError",
    "IsoLossConfig", "ParseError", "Ray", "RenderConfig", "RenderStats", "Scene",
    "ValidationError", "aabb_of", "ellipsoid_volume", "eval_fields", "eval_radiance",
    "gen_test_scene", "iso_scale", "isotropic_loss", "load_cameras", "load_scene", "march_ray",
    "psnr", "ratio_upper_bound", "reference_integrate", "reference_render", "render_image",
    "reorder_by_morton", "save_cameras", "save_scene", "segment_step", "volume_ratio",
    # device-resident / training / ingestion additions
    "DensifyConfig", "GradAccumulator", "MarchLog", "clip_ray_to_scene", "criterion_new",
    "criterion_old", "eval_fields_batch", "load_ply_scene", "look_at_camera", "march_rays",
    "neighbor_density", "observe_scene", "orbit_cameras", "ply_records", "quat_to_rotation",
    "reference_rays", "render", "render_backward", "render_full", "sh_basis", "TraversalOverflow",
    "VARIANTS", "autotune", "fd_position_gradient",
]
