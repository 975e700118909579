"""Morton ordering and BVH queries on the device (spatial.py of the reference).

Bit-exact with the reference: Morton codes (fp64 quantization), the stable
sort permutation, and per-segment candidate SETS (fp64 slab tests on the fp64
AABBs).  Closest hits agree to ~1e-12 (fp64 Kahan quadratic)."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr, stream_ptr
from .errors import BufferOverflow

MORTON_BITS = 21
MORTON_MAX = (1 << MORTON_BITS) - 1


def _dev(device=None):
    return torch.device(device if device is not None else "cuda")


def morton_encode(p, device=None):
    """spatial.py:48-64: (3,) -> int or (N,3) -> uint64 array."""
    L = _lib.lib()
    arr = np.asarray(p)
    single = arr.ndim == 1
    arr = np.ascontiguousarray(np.atleast_2d(arr), dtype=np.int64)
    dev = _dev(device)
    q = torch.as_tensor(arr, device=dev)
    codes = torch.empty(arr.shape[0], dtype=torch.int64, device=dev)
    st = _lib.new_status(dev)
    check(L.gsx_morton_encode(ptr(q), arr.shape[0], ptr(codes), ptr(st), stream_ptr()), "encode")
    try:
        _lib.raise_status(st, "morton_encode")
    except ValueError:
        raise ValueError(f"coordinates must be in [0, 2^{MORTON_BITS})")
    out = codes.cpu().numpy().view(np.uint64)
    return int(out[0]) if single else out


def morton_decode(code, device=None):
    """spatial.py:67-78."""
    L = _lib.lib()
    c = np.ascontiguousarray(np.atleast_1d(np.asarray(code, dtype=np.uint64))).view(np.int64)
    dev = _dev(device)
    ct = torch.as_tensor(c, device=dev)
    q = torch.empty((c.shape[0], 3), dtype=torch.int64, device=dev)
    check(L.gsx_morton_decode(ptr(ct), c.shape[0], ptr(q), stream_ptr()), "decode")
    out = q.cpu().numpy()
    return out[0] if out.shape[0] == 1 and np.ndim(code) == 0 else out


def morton_codes(points, lo, hi, device=None) -> np.ndarray:
    """morton_encode(quantize_points(points, lo, hi)) on the device (fp64 exact)."""
    L = _lib.lib()
    dev = _dev(device)
    pts = torch.as_tensor(np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3), device=dev)
    b = torch.as_tensor(np.concatenate([np.asarray(lo, float).reshape(3),
                                        np.asarray(hi, float).reshape(3)]), device=dev)
    n = pts.shape[0]
    codes = torch.empty(n, dtype=torch.int64, device=dev)
    check(L.gsx_morton_codes(ptr(pts), n, ptr(b[:3]), ptr(b[3:]), ptr(codes), stream_ptr()),
          "morton_codes")
    return codes.cpu().numpy().view(np.uint64)


def sort_codes(codes, device=None):
    """Stable radix sort of uint64 keys: (sorted keys, permutation)."""
    L = _lib.lib()
    dev = _dev(device)
    k = torch.as_tensor(np.ascontiguousarray(codes, dtype=np.uint64).view(np.int64), device=dev)
    n = k.shape[0]
    ko = torch.empty_like(k)
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    ws = torch.empty(L.gsx_sort_workspace_bytes(n), dtype=torch.uint8, device=dev)
    check(L.gsx_sort_codes(ptr(k), n, ptr(ko), ptr(perm), ptr(ws), stream_ptr()), "sort")
    return ko.cpu().numpy().view(np.uint64), perm.cpu().numpy()


def morton_order(points, lo, hi, device=None) -> np.ndarray:
    """spatial.py:89-92: stable permutation sorting points by Z-order code."""
    return sort_codes(morton_codes(points, lo, hi, device), device)[1]


def _queries(o, d, t0, t1):
    return np.concatenate([np.asarray(o, float).reshape(3), np.asarray(d, float).reshape(3),
                           [float(t0), float(t1)]])


def collect_segments(scene, queries, capacity: int):
    """Batched Bvh.segment_overlaps: queries [M,8] (o,d,t0,t1).  Returns
    (counts (M,), idx (M, capacity) sorted ascending storage index, valid up to
    min(count, capacity))."""
    L = _lib.lib()
    dev = scene.device
    q = torch.as_tensor(np.ascontiguousarray(queries, dtype=np.float64).reshape(-1, 8), device=dev)
    m = q.shape[0]
    counts = torch.empty(m, dtype=torch.int64, device=dev)
    idx = torch.full((m, capacity), -1, dtype=torch.int64, device=dev)
    st = _lib.new_status(dev)
    check(L.gsx_collect_segments(ptr(scene.arena), ptr(scene.bvh_arena), scene.n, ptr(q), m,
                                 int(capacity), ptr(counts), ptr(idx), ptr(st), stream_ptr()),
          "collect")
    return counts.cpu().numpy(), idx.cpu().numpy(), st.cpu().numpy()


def segment_overlaps(scene, origin, direction, t0, t1, capacity: int = 64) -> np.ndarray:
    """spatial.py:215-247: candidate storage indices (ascending); raises
    BufferOverflow beyond `capacity`."""
    counts, idx, st = collect_segments(scene, _queries(origin, direction, t0, t1)[None], capacity)
    if counts[0] > capacity:
        raise BufferOverflow(int(counts[0]), capacity)
    return idx[0, :counts[0]].copy()


def closest_hits(scene, queries) -> np.ndarray:
    """Batched closest_hit; NaN where the reference returns None."""
    L = _lib.lib()
    dev = scene.device
    q = torch.as_tensor(np.ascontiguousarray(queries, dtype=np.float64).reshape(-1, 8), device=dev)
    m = q.shape[0]
    t = torch.empty(m, dtype=torch.float64, device=dev)
    check(L.gsx_closest_hit(ptr(scene.arena), ptr(scene.bvh_arena), scene.n, ptr(q), m, ptr(t),
                            stream_ptr()), "closest_hit")
    return t.cpu().numpy()


def closest_hit(scene, origin, direction, t_lo: float, t_hi: float):
    """spatial.py:309-354: smallest ellipsoid entry in [t_lo, t_hi] or None."""
    t = closest_hits(scene, _queries(origin, direction, t_lo, t_hi)[None])[0]
    return None if np.isnan(t) else float(t)


def bvh_export(scene):
    """Topology and boxes of the LBVH (tests)."""
    L = _lib.lib()
    dev = scene.device
    n = scene.n
    m = max(n - 1, 1)
    boxes = torch.empty((m, 2, 2, 3), dtype=torch.float32, device=dev)
    children = torch.empty((m, 2), dtype=torch.int32, device=dev)
    parents = torch.empty(max(2 * n - 1, 2), dtype=torch.int32, device=dev)
    check(L.gsx_bvh_export(ptr(scene.bvh_arena), n, ptr(boxes), ptr(children), ptr(parents),
                           stream_ptr()), "bvh_export")
    return boxes.cpu().numpy(), children.cpu().numpy(), parents.cpu().numpy()
