"""Device-resident scene: the GPU counterpart of the reference `Scene`
(scene.py:24-105).

Storage is the 87-float record layout (scene_io.py:26-44) as a float32
[N, 87] CUDA tensor in storage order, plus `uids` (storage -> stable
identity, scene.py:45).  `_rebuild` runs the device build pipeline

    K1 gsx_prepare            derived SoA + fp64 AABBs + scene bounds
    K2 gsx_morton_codes       fp64-exact 63-bit codes in the scene AABB
    K3 gsx_sort_codes         stable radix sort -> Morton permutation
    K5 gsx_bvh_build          Karras LBVH + refit over that permutation

every time the parameters change (the reference rebuilds its SAH tree in the
same places: construction, apply_permutation, with_mean).
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr, stream_ptr
from .errors import EmptyScene, ParseError, ValidationError

NREC = 87
DEFAULT_SIGMA_EPS = 0.01  # scene.py:21


def _records_from_objects(shapes, coeffs) -> np.ndarray:
    """Pack reference-style GaussianShape / AppearanceCoeffs objects."""
    rows = []
    for s, c in zip(shapes, coeffs):
        rows.append(np.concatenate([
            np.asarray(s.mean, float).reshape(3), np.asarray(s.quat, float).reshape(4),
            np.asarray(s.scales, float).reshape(3), [float(s.sigma)],
            np.asarray(c.sh, float).ravel(), np.asarray(c.sg_axis, float).ravel(),
            np.asarray(c.sg_sharp, float).ravel(), np.asarray(c.sg_amp, float).ravel()]))
    return np.stack(rows)


class Scene:
    """GPU scene.  Construct from records (`Scene.from_records`) or, like the
    reference, from lists of shape / appearance objects."""

    def __init__(self, shapes=None, coeffs=None, sigma_eps: float = DEFAULT_SIGMA_EPS, *,
                 records=None, device=None, uids=None):
        if records is None:
            if shapes is None or len(shapes) == 0:
                raise EmptyScene("scene needs at least one primitive")
            if coeffs is None or len(shapes) != len(coeffs):
                raise ValidationError("shape/appearance count mismatch")
            records = _records_from_objects(shapes, coeffs)
        if sigma_eps <= 0:
            raise ValidationError("sigma_eps must be positive")
        L = _lib.lib()
        self.device = torch.device(device if device is not None else "cuda")
        if isinstance(records, torch.Tensor):
            params = records.detach().to(device=self.device, dtype=torch.float32)
        else:
            params = torch.as_tensor(np.asarray(records, dtype=np.float32), device=self.device)
        params = params.reshape(-1, NREC).contiguous()
        if params.shape[0] == 0:
            raise EmptyScene("scene needs at least one primitive")
        self._L = L
        self.params = params
        self.sigma_eps = float(sigma_eps)
        n = params.shape[0]
        if uids is None:
            self.uids_t = torch.arange(n, dtype=torch.int64, device=self.device)
        else:
            self.uids_t = torch.as_tensor(uids, dtype=torch.int64, device=self.device).clone()
        self._alloc(n)
        self._rebuild()

    @classmethod
    def from_records(cls, records, sigma_eps: float = DEFAULT_SIGMA_EPS, device=None) -> "Scene":
        return cls(records=records, sigma_eps=sigma_eps, device=device)

    # -- buffers -----------------------------------------------------------
    def _alloc(self, n: int):
        L, dev = self._L, self.device
        u8 = torch.uint8
        self.n = n
        self.arena = torch.empty(L.gsx_scene_arena_bytes(n), dtype=u8, device=dev)
        self.bvh_arena = torch.empty(L.gsx_bvh_arena_bytes(n), dtype=u8, device=dev)
        self._sort_ws = torch.empty(L.gsx_sort_workspace_bytes(n), dtype=u8, device=dev)
        self._bvh_ws = torch.empty(L.gsx_bvh_workspace_bytes(n), dtype=u8, device=dev)
        self._codes = torch.empty(n, dtype=torch.int64, device=dev)  # u64 bit pattern
        self.sorted_codes = torch.empty(n, dtype=torch.int64, device=dev)
        self.morton_perm = torch.empty(n, dtype=torch.int64, device=dev)
        self.bounds_t = torch.empty(6, dtype=torch.float64, device=dev)
        self._status = _lib.new_status(dev)

    def render_status(self):
        """Sticky device status word of this scene's renders (traversal-stack
        overflow, GSX_ERR_STACK): written by the kernels, read -- and the
        error raised -- only by check_render_status(), so renders stay
        asynchronous."""
        st = getattr(self, "_render_st", None)
        if st is None:
            st = _lib.new_status(self.device)
            self._render_st = st
        return st

    def check_render_status(self):
        """Raise TraversalOverflow if any render / backward of this scene since
        the last check overflowed a traversal stack (synchronizes), then clear."""
        st = self.render_status()
        try:
            _lib.raise_status(st, "render")
        finally:
            st.copy_(_lib.new_status(self.device))

    def render_workspace(self):
        """The scene's default per-render workspace (gsx_render_workspace_bytes:
        the per-camera silhouette table of the screened forward)."""
        ws = getattr(self, "_render_ws", None)
        need = int(self._L.gsx_render_workspace_bytes(self.n))
        if ws is None or ws.numel() < need:
            ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            self._render_ws = ws
        return ws

    def _rebuild(self, validate: bool = True):
        """K1 -> K2 -> K3 -> K5 (see module docstring)."""
        L, n, s = self._L, self.n, stream_ptr()
        self.version = getattr(self, "version", 0) + 1
        self._status.copy_(_lib.new_status(self.device))
        hb = (torch.empty(6, dtype=torch.float64)).numpy()
        check(L.gsx_prepare(ptr(self.params), n, self.sigma_eps, ptr(self.arena),
                            ptr(self._status), hb.ctypes.data_as(_lib.P), s), "prepare")
        if validate:
            _lib.raise_status(self._status, "prepare")
        self.bounds_lo = hb[:3].copy()
        self.bounds_hi = hb[3:].copy()
        self.bounds_t.copy_(torch.from_numpy(hb))
        bl = self.bounds_t[:3]
        bh = self.bounds_t[3:]
        check(L.gsx_morton_codes_records(ptr(self.params), n, ptr(bl), ptr(bh), ptr(self._codes),
                                         s), "morton")
        check(L.gsx_sort_codes(ptr(self._codes), n, ptr(self.sorted_codes), ptr(self.morton_perm),
                               ptr(self._sort_ws), s), "sort")
        check(L.gsx_bvh_build(ptr(self.arena), ptr(self.sorted_codes), ptr(self.morton_perm), n,
                              ptr(self.bvh_arena), ptr(self._bvh_ws), s), "bvh")

    def rebuild(self):
        """Re-derive everything after `params` was updated in place (training)."""
        self._rebuild(validate=True)

    def rebuild_async(self):
        """K1 -> K5 without any host synchronization (training hot loop): the
        scene bounds stay on the device; validation errors are not raised
        (the optimizer's projection keeps records valid)."""
        L, n, s = self._L, self.n, stream_ptr()
        self.version = getattr(self, "version", 0) + 1
        check(L.gsx_prepare(ptr(self.params), n, self.sigma_eps, ptr(self.arena),
                            ptr(self._status), None, s), "prepare")
        check(L.gsx_scene_get(ptr(self.arena), n, 4, ptr(self.bounds_t), s), "bounds")
        bl, bh = self.bounds_t[:3], self.bounds_t[3:]
        check(L.gsx_morton_codes_records(ptr(self.params), n, ptr(bl), ptr(bh), ptr(self._codes),
                                         s), "morton")
        check(L.gsx_sort_codes(ptr(self._codes), n, ptr(self.sorted_codes), ptr(self.morton_perm),
                               ptr(self._sort_ws), s), "sort")
        check(L.gsx_bvh_build(ptr(self.arena), ptr(self.sorted_codes), ptr(self.morton_perm), n,
                              ptr(self.bvh_arena), ptr(self._bvh_ws), s), "bvh")

    def rebuild_graphed(self):
        """rebuild_async replayed from a CUDA graph (captured on first use, per
        parameter buffer): the ~40 launches of K1-K5 (prepare, bounds,
        Morton codes, 8 radix passes, Karras, refit, the cooperative 4-wide
        collapse) go to the GPU as one graph launch.  Falls back to eager
        launches if the capture fails."""
        key = (self.params.data_ptr(), self.n)
        g = getattr(self, "_rebuild_graph", None)
        if g is None or getattr(self, "_rebuild_key", None) != key:
            g = None
            if not getattr(self, "_rebuild_no_graph", False):
                try:
                    self.rebuild_async()  # warm-up outside the capture
                    torch.cuda.current_stream().synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        self.rebuild_async()
                except Exception:  # (capture unsupported here: eager from now on)
                    self._rebuild_no_graph = True
                    g = None
            self._rebuild_graph, self._rebuild_key = g, key
        if g is None:
            self.rebuild_async()
            return
        g.replay()
        self.version = getattr(self, "version", 0) + 1

    # -- reference API -------------------------------------------------------
    def __len__(self) -> int:
        return self.n

    @property
    def uids(self) -> np.ndarray:
        return self.uids_t.cpu().numpy()

    def apply_permutation(self, perm):
        """scene.py:74-80: permute primitive storage and rebuild."""
        perm_t = torch.as_tensor(np.asarray(perm, dtype=np.int64) if not isinstance(
            perm, torch.Tensor) else perm, dtype=torch.int64, device=self.device).contiguous()
        out = torch.empty_like(self.params)
        uids = torch.empty_like(self.uids_t)
        check(self._L.gsx_permute(ptr(self.params), ptr(self.uids_t), ptr(perm_t), self.n,
                                  ptr(out), ptr(uids), stream_ptr()), "permute")
        self.params = out
        self.uids_t = uids
        self._rebuild()

    def with_mean(self, index: int, mean) -> "Scene":
        """scene.py:82-94: copy with one primitive's mean replaced."""
        rec = self.params.clone()
        rec[index, 0:3] = torch.as_tensor(np.asarray(mean, dtype=np.float32), device=self.device)
        return Scene(records=rec, sigma_eps=self.sigma_eps, device=self.device,
                     uids=self.uids_t)

    def records(self) -> np.ndarray:
        return self.params.detach().cpu().numpy().astype(np.float64)

    @property
    def means(self) -> np.ndarray:
        return self.records()[:, 0:3]

    def _get(self, which: int, shape) -> np.ndarray:
        out = torch.empty(int(np.prod(shape)), dtype=torch.float64, device=self.device)
        check(self._L.gsx_scene_get(ptr(self.arena), self.n, which, ptr(out), stream_ptr()),
              "scene_get")
        return out.cpu().numpy().reshape(shape)

    @property
    def aabb_lo(self) -> np.ndarray:
        return self._get(0, (self.n, 3))

    @property
    def aabb_hi(self) -> np.ndarray:
        return self._get(1, (self.n, 3))

    @property
    def iso_inv(self) -> np.ndarray:
        return self._get(2, (self.n, 3, 3))

    @property
    def log_ratio(self) -> np.ndarray:
        return self._get(3, (self.n,))

    def morton_codes(self) -> np.ndarray:
        """Codes of the current storage order (uint64), quantized in the scene AABB."""
        return self._codes.cpu().numpy().view(np.uint64)


def reorder_by_morton(scene: Scene) -> np.ndarray:
    """scene.py:97-105: sort storage by ascending Z-order code of the means
    (bit-exact codes and stable permutation); returns the applied permutation."""
    perm = scene.morton_perm.clone()
    scene.apply_permutation(perm)
    return perm.cpu().numpy()


# -- .gsx I/O (scene_io.py:25-108) ----------------------------------------------
GSX_VERSION = 1


def save_scene(scene: Scene, path):
    path = Path(path)
    rec = scene.params.detach().cpu().numpy().astype("<f4")
    path.write_bytes(rec.tobytes())
    header = {"format": "gsx", "version": GSX_VERSION, "sigma_eps": scene.sigma_eps,
              "count": len(scene), "floats_per_record": NREC}
    Path(str(path) + ".json").write_text(json.dumps(header, indent=2) + "\n")


def load_records(path):
    """(records float32 [N,87], sigma_eps) from a .gsx file + JSON sidecar."""
    path = Path(path)
    sidecar = Path(str(path) + ".json")
    if not path.exists() or not sidecar.exists():
        raise ParseError(f"missing scene file or sidecar header for {path}")
    try:
        header = json.loads(sidecar.read_text())
    except json.JSONDecodeError as e:
        raise ParseError(f"bad sidecar header: {e}") from e
    if header.get("format") != "gsx" or header.get("version") != GSX_VERSION:
        raise ParseError(f"unsupported scene format header: {header}")
    count = int(header.get("count", -1))
    if count <= 0:
        raise ValidationError("scene must contain at least one primitive")
    if int(header.get("floats_per_record", -1)) != NREC:
        raise ParseError("record layout mismatch")
    raw = np.frombuffer(path.read_bytes(), dtype="<f4")
    if raw.size != count * NREC:
        raise ParseError(f"expected {count * NREC} floats, found {raw.size}")
    return raw.reshape(count, NREC), float(header["sigma_eps"])


def load_scene(path, reorder: bool = False, device=None) -> Scene:
    rec, eps = load_records(path)
    scene = Scene(records=rec, sigma_eps=eps, device=device)
    if reorder:
        reorder_by_morton(scene)
    return scene


def gen_test_scene(kind: str = "random-cloud", count: int = 32, seed: int = 0,
                   anisotropy: float = 1.0, sigma_eps: float = DEFAULT_SIGMA_EPS,
                   extent: float = 1.0, base_scale: float = 0.08, device=None) -> Scene:
    """scene_io.py:206-273 on the device (same records as the reference
    generator, rounded to float32)."""
    from .scenes import gen_test_scene_records

    rec = gen_test_scene_records(kind, count, seed, anisotropy, extent, base_scale)
    return Scene(records=rec.astype(np.float32), sigma_eps=sigma_eps, device=device)
