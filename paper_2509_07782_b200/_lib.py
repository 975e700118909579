"""ctypes binding of libgsx.so (the C ABI declared in include/gsx.h).

The library is built in-tree (`paper_2509_07782_b200/libgsx.so`, see
csrc/Makefile or `__graft_entry__.build()`).  There is no fallback: if the
library or a CUDA device is missing, every entry point raises
`GsxUnavailable` -- the product path never silently degrades to CPU code.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

from .errors import BufferOverflow, EmptyScene, GsrayError, TraversalOverflow, ValidationError

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libgsx.so"
CSRC = _HERE / "csrc"

GSX_OK, GSX_ERR_EMPTY, GSX_ERR_VALIDATION, GSX_ERR_OVERFLOW, GSX_ERR_ARG, GSX_ERR_CUDA, \
    GSX_ERR_STACK = range(7)

INT64_MAX = (1 << 63) - 1


class GsxUnavailable(GsrayError):
    """libgsx.so or a CUDA device is missing (no CPU fallback exists)."""


class GsxCudaError(GsrayError):
    """A CUDA launch or runtime call inside libgsx failed."""


class RenderCfg(ctypes.Structure):
    _fields_ = [
        ("dt", ctypes.c_double), ("n_s", ctypes.c_int64), ("t_eps", ctypes.c_double),
        ("mode", ctypes.c_int64), ("beta", ctypes.c_double), ("dt_min", ctypes.c_double),
        ("dt_max", ctypes.c_double), ("ess", ctypes.c_int64), ("tile_size", ctypes.c_int64),
        ("background", ctypes.c_double * 3), ("buffer_capacity", ctypes.c_int64),
        ("traversal", ctypes.c_int64), ("sums", ctypes.c_int64), ("pass2", ctypes.c_int64),
    ]


class CameraC(ctypes.Structure):
    _fields_ = [
        ("R", ctypes.c_double * 9), ("center", ctypes.c_double * 3), ("focal", ctypes.c_double),
        ("width", ctypes.c_int64), ("height", ctypes.c_int64), ("t_near", ctypes.c_double),
        ("t_far", ctypes.c_double),
    ]


class Stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in (
        "rays", "samples", "segments", "segments_skipped", "closest_hit_calls", "node_visits",
        "aabb_hits", "ellipsoid_hits", "pairs", "composited")]


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile libgsx.so for sm_100a with nvcc (csrc/Makefile)."""
    args = ["make", "-C", str(CSRC), "-j8"]
    if force:
        subprocess.run(["make", "-C", str(CSRC), "clean"], check=True, capture_output=True)
    res = subprocess.run(args, capture_output=not verbose, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"libgsx build failed:\n{res.stdout}\n{res.stderr}")
    return LIB_PATH


_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
D = ctypes.c_double
SZ = ctypes.c_size_t
INT = ctypes.c_int

_SIGS = {
    "gsx_status_string": (ctypes.c_char_p, [INT]),
    "gsx_abi_version": (INT, []),
    "gsx_last_cuda_error": (ctypes.c_char_p, []),
    "gsx_scene_arena_bytes": (SZ, [I64]),
    "gsx_prepare": (INT, [P, I64, D, P, P, P, P]),
    "gsx_scene_get": (INT, [P, I64, INT, P, P]),
    "gsx_morton_codes": (INT, [P, I64, P, P, P, P]),
    "gsx_morton_codes_records": (INT, [P, I64, P, P, P, P]),
    "gsx_morton_encode": (INT, [P, I64, P, P, P]),
    "gsx_morton_decode": (INT, [P, I64, P, P]),
    "gsx_sort_workspace_bytes": (SZ, [I64]),
    "gsx_sort_codes": (INT, [P, I64, P, P, P, P]),
    "gsx_permute": (INT, [P, P, P, I64, P, P, P]),
    "gsx_bvh_arena_bytes": (SZ, [I64]),
    "gsx_bvh_workspace_bytes": (SZ, [I64]),
    "gsx_bvh_build": (INT, [P, P, P, I64, P, P, P]),
    "gsx_bvh_export": (INT, [P, I64, P, P, P, P]),
    "gsx_bvh_collapse": (INT, [P, I64, P, P]),
    "gsx_collect_segments": (INT, [P, P, I64, P, I64, I64, P, P, P, P]),
    "gsx_closest_hit": (INT, [P, P, I64, P, I64, P, P]),
    "gsx_render_workspace_bytes": (SZ, [I64]),
    "gsx_tile_id": (I64, [I64, I64, I64, I64]),
    "gsx_render_forward": (INT, [P, P, I64, P, P, I64, I64, P, P, P, P, P, I64, P, P]),
    "gsx_render_rays": (INT, [P, P, I64, P, I64, INT, P, P, P, P, P, P, P]),
    "gsx_render_rays_stats": (INT, [P, P, I64, P, I64, INT, P, P, P, P, P, P, P]),
    "gsx_render_backward": (INT, [P, P, P, I64, P, P, I64, I64, P, P, P, P, P, P, P, P, P]),
    "gsx_march_log_min_bytes": (I64, [P, I64, I64]),
    "gsx_render_forward_logged": (INT, [P, P, I64, P, P, I64, I64, P, P, P, P, I64, P, I64, P,
                                        P]),
    "gsx_render_backward_logged": (INT, [P, P, P, I64, P, P, I64, I64, P, P, P, P, P, P, P, P,
                                         P, P]),
    "gsx_march_log_usage": (INT, [P, P, P, P]),
    "gsx_densify_observe": (INT, [P, P, I64, P, I64, P, D, P, P, P, P]),
    "gsx_neighbor_density": (INT, [P, P, I64, D, P, P, P]),
    "gsx_densify_criteria": (INT, [P, P, P, I64, D, P, P, P]),
    "gsx_calibrate_fp32": (INT, [I64, P, P, P]),
    "gsx_calibrate_sfu": (INT, [I64, P, P, P]),
    "gsx_reference_rays": (INT, [P, P, I64, P, I64, INT, D, P, P, P]),
    "gsx_eval_fields": (INT, [P, P, I64, P, P, I64, P, I64, P, P, P, P]),
    "gsx_image_loss_workspace_bytes": (SZ, [I64, I64, I64]),
    "gsx_image_loss": (INT, [P, P, I64, I64, I64, D, P, P, P, P]),
    "gsx_iso_loss": (INT, [P, I64, D, D, P, P, P]),
    "gsx_adam_step": (INT, [P, P, P, P, I64, P, P, D, D, D, I64, P]),
}

# Every symbol include/gsx.h declares (checked by tests/test_abi.py).
EXPORTED = tuple(_SIGS)


def load_library(path: Path | None = None):
    """Load libgsx.so without touching CUDA (symbol checks work on CPU hosts)."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("GSX_LIB", LIB_PATH))
    if not p.exists():
        raise GsxUnavailable(f"{p} not built; run __graft_entry__.build() (nvcc, sm_100a)")
    L = ctypes.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def lib():
    """The library, after checking a CUDA device is present."""
    import torch

    L = load_library()
    if not torch.cuda.is_available():
        raise GsxUnavailable("no CUDA device: the gsx render path has no CPU fallback")
    return L


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def check(rc: int, what: str = ""):
    if rc == GSX_OK:
        return
    L = load_library()
    msg = L.gsx_status_string(rc).decode()
    if rc == GSX_ERR_CUDA:
        raise GsxCudaError(f"{what}: {msg}: {L.gsx_last_cuda_error().decode()}")
    if rc == GSX_ERR_EMPTY:
        raise EmptyScene(f"{what}: {msg}")
    if rc == GSX_ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    if rc == GSX_ERR_VALIDATION:
        raise ValidationError(f"{what}: {msg}")
    if rc == GSX_ERR_STACK:
        raise TraversalOverflow(f"{what}: {msg}")
    raise GsrayError(f"{what}: {msg} (status {rc})")


def new_status(device):
    import torch

    return torch.tensor([0, INT64_MAX, 0, 0], dtype=torch.int64, device=device)


def raise_status(st, what: str = ""):
    """Read a device status word (synchronizes) and raise the mapped error."""
    code, index, count, cap = (int(x) for x in st.tolist())
    if code == GSX_OK:
        return
    if code == GSX_ERR_VALIDATION:
        raise ValidationError(f"{what}: invalid primitive record", record=index)
    if code == GSX_ERR_OVERFLOW:
        raise BufferOverflow(count, cap)
    if code == GSX_ERR_ARG:
        raise ValueError(f"{what}: argument out of range at {index}")
    if code == GSX_ERR_STACK:
        raise TraversalOverflow(f"{what}: traversal stack overflow (pixel / ray {index})", index)
    check(code, what)
