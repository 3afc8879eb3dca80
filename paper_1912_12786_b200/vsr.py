"""Thin ctypes binding over libvsr.so (include/vsr.h) — argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind ``vsr_trace``; this
module only converts Python/numpy/torch arguments into the C ABI's plain
pointers and sizes.  There is no CPU fallback: if ``libvsr.so`` is missing the
import of :func:`lib` raises.  PyTorch is used for device memory and streams
only (``torch.Tensor.data_ptr()``, ``torch.cuda.current_stream().cuda_stream``).
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VSR_LIB") or os.path.join(_HERE, "libvsr.so")   # VSR_LIB: tuning builds

# vsr_status
OK, ERR_INVALID_ARG, ERR_EMPTY_SCENE, ERR_NONFINITE, ERR_BVH_TOO_DEEP, ERR_NOT_BUILT, \
    ERR_CUDA, ERR_OOM, ERR_UNSUPPORTED = range(9)
STATUS_NAMES = ["VSR_OK", "VSR_ERR_INVALID_ARG", "VSR_ERR_EMPTY_SCENE", "VSR_ERR_NONFINITE",
                "VSR_ERR_BVH_TOO_DEEP", "VSR_ERR_NOT_BUILT", "VSR_ERR_CUDA", "VSR_ERR_OOM",
                "VSR_ERR_UNSUPPORTED"]
# vsr_query
CLOSEST, ANY = 0, 1
# vsr_isect
NONE, DEFAULT, ALPHA_TEXTURE, ALPHA_PROCEDURAL, COUNT, COUNT_ALPHA_TEXTURE = range(6)
ALPHA_TEXTURE_BILINEAR, ALPHA_PROCEDURAL_UV = 6, 7   # NEXT-4 sampling variants
RUNTIME_SWITCH_DEFAULT, RUNTIME_SWITCH_ALPHA_TEXTURE, RUNTIME_SWITCH_ALPHA_PROCEDURAL = 101, 102, 103
RUNTIME_FNPTR_DEFAULT, RUNTIME_FNPTR_ALPHA_TEXTURE, RUNTIME_FNPTR_ALPHA_PROCEDURAL = 201, 202, 203
ISECT_NAMES = {NONE: "none", DEFAULT: "default", ALPHA_TEXTURE: "alpha_texture",
               ALPHA_PROCEDURAL: "alpha_procedural", COUNT: "count",
               COUNT_ALPHA_TEXTURE: "count_alpha_texture",
               ALPHA_TEXTURE_BILINEAR: "alpha_texture_bilinear",
               ALPHA_PROCEDURAL_UV: "alpha_procedural_uv",
               RUNTIME_SWITCH_DEFAULT: "runtime_switch_default",
               RUNTIME_SWITCH_ALPHA_TEXTURE: "runtime_switch_alpha_texture",
               RUNTIME_SWITCH_ALPHA_PROCEDURAL: "runtime_switch_alpha_procedural",
               RUNTIME_FNPTR_DEFAULT: "runtime_fnptr_default",
               RUNTIME_FNPTR_ALPHA_TEXTURE: "runtime_fnptr_alpha_texture",
               RUNTIME_FNPTR_ALPHA_PROCEDURAL: "runtime_fnptr_alpha_procedural"}
MISS = 0xFFFFFFFF

HIT_DTYPE = np.dtype([("t", "<f4"), ("u", "<f4"), ("v", "<f4"), ("prim", "<u4")])
COUNTS_DTYPE = np.dtype([("boxes", "<u4"), ("tris", "<u4"), ("alpha", "<u4"), ("reserved", "<u4")])

EXPORTED_SYMBOLS = ["vsr_scene_create", "vsr_bvh_build", "vsr_trace", "vsr_trace_multi",
                    "vsr_trace_host",
                    "vsr_destroy", "vsr_last_error", "vsr_bvh_export", "vsr_scene_import",
                    "vsr_scene_stats", "vsr_launch_count", "vsr_abi_version",
                    "vsr_set_kernel_events", "vsr_group_create", "vsr_group_destroy",
                    "vsr_trace_group", "vsr_instances_create", "vsr_instances_destroy",
                    "vsr_trace_instances", "vsr_instances_export", "vsr_bvh_build_gpu",
                    "vsr_trace_pinhole", "vsr_trace_tiles", "vsr_device_alloc", "vsr_device_free",
                    "vsr_ipc_handle", "vsr_ipc_open", "vsr_ipc_close", "vsr_bvh_build_ploc",
                    "vsr_trace_group_multi", "vsr_trace_instances_multi", "vsr_trace_primitives",
                    "vsr_bvh8_build", "vsr_bvh8_export", "vsr_trace_bvh8"]


class VsrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {msg}")


class TextureDesc(C.Structure):
    _fields_ = [("width", C.c_uint32), ("height", C.c_uint32), ("rgba8", C.c_void_p)]


class SceneDesc(C.Structure):
    _fields_ = [("num_tris", C.c_uint32), ("vertices", C.c_void_p), ("geom_ids", C.c_void_p),
                ("texcoords", C.c_void_p), ("num_geoms", C.c_uint32),
                ("geom_texture", C.c_void_p), ("num_textures", C.c_uint32),
                ("textures", C.c_void_p), ("device", C.c_int)]


class BuildParams(C.Structure):
    _fields_ = [("max_leaf_size", C.c_uint32), ("sah_bins", C.c_uint32),
                ("traversal_cost", C.c_float), ("intersection_cost", C.c_float)]


class IsectParams(C.Structure):
    _fields_ = [("alpha_threshold", C.c_float), ("checker_freq", C.c_uint32)]


class Bvh8View(C.Structure):
    _fields_ = [("num_nodes", C.c_uint32), ("num_tris", C.c_uint32), ("max_depth", C.c_uint32),
                ("pad", C.c_uint32), ("root_lo", C.c_float * 3), ("root_hi", C.c_float * 3),
                ("build_ms", C.c_double), ("nodes", C.c_void_p), ("tris", C.c_void_p),
                ("sides", C.c_void_p)]


class BvhView(C.Structure):
    _fields_ = [("root_ref", C.c_uint32), ("root_lo", C.c_float * 3), ("root_hi", C.c_float * 3),
                ("num_nodes", C.c_uint32), ("num_tris", C.c_uint32), ("num_textures", C.c_uint32),
                ("num_texels", C.c_uint64), ("nodes", C.c_void_p), ("tris", C.c_void_p),
                ("sides", C.c_void_p), ("texdescs", C.c_void_p), ("texels", C.c_void_p)]


class Instance(C.Structure):
    _fields_ = [("bvh", C.c_uint32), ("object_from_world", C.c_float * 12)]


class InstancesView(C.Structure):
    _fields_ = [("root_ref", C.c_uint32), ("root_lo", C.c_float * 3), ("root_hi", C.c_float * 3),
                ("num_nodes", C.c_uint32), ("num_instances", C.c_uint32),
                ("max_depth", C.c_uint32), ("r_safe", C.c_float), ("nodes", C.c_void_p),
                ("records", C.c_void_p)]


class Pinhole(C.Structure):
    _fields_ = [("eye", C.c_double * 3), ("w", C.c_double * 3), ("u", C.c_double * 3),
                ("v", C.c_double * 3), ("tan_half_vfov", C.c_double), ("aspect", C.c_double),
                ("width", C.c_uint32), ("height", C.c_uint32), ("spp", C.c_uint32),
                ("jitter_seed", C.c_uint32), ("tmin", C.c_float), ("tmax", C.c_float)]


def pinhole_camera(eye, look_at, up, vfov_deg, width, height, spp=1, jitter_seed=6, tmin=1e-4,
                   tmax=float("inf")) -> Pinhole:
    """vsr_pinhole for a look-at camera: w = normalize(look_at - eye), u = normalize(up x w),
    v = w x u, all in fp64 (the input recipe's basis)."""
    e = np.asarray(eye, dtype=np.float64)
    w = np.asarray(look_at, dtype=np.float64) - e
    w /= np.linalg.norm(w)
    u = np.cross(np.asarray(up, dtype=np.float64), w)
    u /= np.linalg.norm(u)
    v = np.cross(w, u)
    c = Pinhole()
    c.eye = (C.c_double * 3)(*e.tolist())
    c.w = (C.c_double * 3)(*w.tolist())
    c.u = (C.c_double * 3)(*u.tolist())
    c.v = (C.c_double * 3)(*v.tolist())
    c.tan_half_vfov = math.tan(math.radians(vfov_deg) * 0.5)
    c.aspect = width / height
    c.width, c.height, c.spp, c.jitter_seed = width, height, spp, jitter_seed
    c.tmin, c.tmax = tmin, tmax
    return c


class Stats(C.Structure):
    _fields_ = [("num_tris_input", C.c_uint32), ("num_tris", C.c_uint32),
                ("num_degenerate", C.c_uint32), ("num_nodes", C.c_uint32),
                ("num_leaves", C.c_uint32), ("max_depth", C.c_uint32),
                ("num_textures", C.c_uint32), ("built", C.c_uint32), ("num_texels", C.c_uint64),
                ("device_bytes", C.c_uint64), ("build_ms", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load libvsr.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.vsr_scene_create.argtypes = [C.POINTER(SceneDesc), C.POINTER(P)]
        L.vsr_bvh_build.argtypes = [P, C.POINTER(BuildParams)]
        L.vsr_bvh_build_gpu.argtypes = [P, C.c_uint32]
        L.vsr_trace_pinhole.argtypes = [P, C.POINTER(Pinhole), C.c_int, C.c_int,
                                        C.POINTER(IsectParams), P, P, P]
        L.vsr_trace_pinhole.restype = C.c_int
        L.vsr_trace_tiles.argtypes = [P, P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                      C.c_int, C.POINTER(IsectParams), P, P, P]
        L.vsr_device_alloc.argtypes = [C.c_uint64, C.c_int, C.POINTER(P)]
        L.vsr_device_free.argtypes = [P, C.c_int]
        L.vsr_ipc_handle.argtypes = [P, P]
        L.vsr_ipc_open.argtypes = [P, C.c_int, C.POINTER(P)]
        L.vsr_ipc_close.argtypes = [P, C.c_int]
        for name in ("vsr_trace_tiles", "vsr_device_alloc", "vsr_device_free", "vsr_ipc_handle",
                     "vsr_ipc_open", "vsr_ipc_close"):
            getattr(L, name).restype = C.c_int
        L.vsr_bvh_build_gpu.restype = C.c_int
        L.vsr_bvh_build_ploc.argtypes = [P, C.c_uint32, C.c_uint32]
        L.vsr_bvh_build_ploc.restype = C.c_int
        L.vsr_bvh8_build.argtypes = [P]
        L.vsr_bvh8_build.restype = C.c_int
        L.vsr_bvh8_export.argtypes = [P, C.POINTER(Bvh8View)]
        L.vsr_bvh8_export.restype = C.c_int
        L.vsr_trace_bvh8.argtypes = [P, P, C.c_uint64, C.c_int, C.c_int, C.POINTER(IsectParams),
                                     P, P, P]
        L.vsr_trace_bvh8.restype = C.c_int
        for name in ("vsr_trace_group_multi", "vsr_trace_instances_multi"):
            getattr(L, name).argtypes = [P, P, C.c_uint64, C.c_uint32, C.c_int,
                                         C.POINTER(IsectParams), P, P, P, P, P]
            getattr(L, name).restype = C.c_int
        L.vsr_trace.argtypes = [P, P, C.c_uint64, C.c_int, C.c_int, C.POINTER(IsectParams), P, P, P]
        L.vsr_trace_host.argtypes = [P, P, C.c_uint64, C.c_int, C.c_int, C.POINTER(IsectParams),
                                     P, P, P]
        L.vsr_trace_primitives.argtypes = [P, P, C.c_uint64, C.c_int, C.c_int,
                                           C.POINTER(IsectParams), P, P, P]
        L.vsr_trace_primitives.restype = C.c_int
        L.vsr_trace_multi.argtypes = [P, P, C.c_uint64, C.c_uint32, C.c_int,
                                      C.POINTER(IsectParams), P, P, P, P]
        L.vsr_destroy.argtypes = [P]
        L.vsr_last_error.restype = C.c_char_p
        L.vsr_bvh_export.argtypes = [P, C.POINTER(BvhView)]
        L.vsr_scene_import.argtypes = [C.POINTER(BvhView), C.c_int, C.POINTER(P)]
        L.vsr_scene_stats.argtypes = [P, C.POINTER(Stats)]
        L.vsr_launch_count.restype = C.c_uint64
        L.vsr_abi_version.restype = C.c_uint32
        L.vsr_set_kernel_events.argtypes = [P, P]
        L.vsr_set_kernel_events.restype = C.c_int
        L.vsr_group_create.argtypes = [P, C.c_uint32, C.POINTER(P)]
        L.vsr_group_destroy.argtypes = [P]
        L.vsr_trace_group.argtypes = [P, P, C.c_uint64, C.c_int, C.c_int, C.POINTER(IsectParams),
                                      P, P, P, P]
        L.vsr_instances_create.argtypes = [P, C.c_uint32, P, C.c_uint32, C.POINTER(BuildParams),
                                           C.POINTER(P)]
        L.vsr_instances_destroy.argtypes = [P]
        L.vsr_instances_export.argtypes = [P, C.POINTER(InstancesView)]
        L.vsr_trace_instances.argtypes = [P, P, C.c_uint64, C.c_int, C.c_int,
                                          C.POINTER(IsectParams), P, P, P, P]
        for name in ("vsr_group_create", "vsr_group_destroy", "vsr_trace_group",
                     "vsr_instances_create", "vsr_instances_destroy", "vsr_instances_export",
                     "vsr_trace_instances"):
            getattr(L, name).restype = C.c_int
        for name in ("vsr_scene_create", "vsr_bvh_build", "vsr_trace", "vsr_trace_multi",
                     "vsr_trace_host",
                     "vsr_destroy", "vsr_bvh_export", "vsr_scene_import", "vsr_scene_stats"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(status: int):
    if status != OK:
        raise VsrError(status, lib().vsr_last_error().decode())


def launch_count() -> int:
    return int(lib().vsr_launch_count())


def set_kernel_events(start=None, stop=None):
    """Profiling hook: record torch.cuda.Event `start`/`stop` around the trace kernel
    itself (after the block-order pass) on this thread; None, None disables."""
    h = lambda e: None if e is None else e.cuda_event  # noqa: E731
    _check(lib().vsr_set_kernel_events(h(start), h(stop)))


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def _stream_handle(stream, device=None):
    """Raw cudaStream_t: the given stream, else the current stream of `device`
    (the scene's device, not whichever device happens to be current)."""
    if stream is None:
        import torch
        return torch.cuda.current_stream(device).cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _check_dev(t, name, dtype, rows, tail, device, optional=False):
    """Argument check before a device pointer crosses the C ABI (the C side only
    sees NULL and alignment): a contiguous CUDA tensor on the scene's device with
    the expected dtype, at least `rows` rows and trailing shape `tail`.  Raises
    ValueError on a mismatch instead of letting a kernel read or write out of bounds."""
    import torch
    if t is None:
        if optional:
            return
        raise ValueError(f"{name}: a CUDA tensor is required")
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name}: expected a torch CUDA tensor, got {type(t).__name__}")
    if not t.is_cuda or (device is not None and t.device.index != device):
        raise ValueError(f"{name}: must live on cuda:{device}, got {t.device}")
    if t.dtype not in dtype:
        raise ValueError(f"{name}: dtype {t.dtype} not in {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if t.dim() != 1 + len(tail) or tuple(t.shape[1:]) != tuple(tail) or t.shape[0] < rows:
        raise ValueError(f"{name}: shape {tuple(t.shape)}, need [>= {rows}, "
                         f"{', '.join(map(str, tail))}]")


def _f32():
    import torch
    return (torch.float32,)


def _i32():
    import torch
    return (torch.int32, torch.uint32) if hasattr(torch, "uint32") else (torch.int32,)


def _check_rays(rays, n, device):
    _check_dev(rays, "rays", _f32(), n, (8,), device)
    if n > rays.shape[0]:
        raise ValueError(f"n={n} exceeds rays.shape[0]={rays.shape[0]}")


def _check_host(a, name, rows, row_bytes):
    """Host buffer for vsr_trace_host: C-contiguous, >= rows x row_bytes bytes."""
    if hasattr(a, "is_cuda"):
        if a.is_cuda or not a.is_contiguous():
            raise ValueError(f"{name}: expected a contiguous host tensor")
        nbytes = a.numel() * a.element_size()
    else:
        if not isinstance(a, np.ndarray) or not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name}: expected a C-contiguous numpy array")
        nbytes = a.nbytes
    if nbytes < rows * row_bytes:
        raise ValueError(f"{name}: {nbytes} bytes, need {rows * row_bytes}")


class Scene:
    """A scene on one device: vsr_scene_create + vsr_bvh_build, then vsr_trace."""

    def __init__(self, vertices=None, geom_ids=None, texcoords=None, geom_texture=None,
                 textures=None, device: int = 0, _handle=None):
        self.device = device
        self._h = C.c_void_p()
        if _handle is not None:
            self._h = _handle
            return
        v = np.ascontiguousarray(vertices, dtype=np.float32).reshape(-1, 9)
        keep = [v]
        g = None if geom_ids is None else np.ascontiguousarray(geom_ids, dtype=np.uint32)
        tc = None if texcoords is None else np.ascontiguousarray(texcoords, dtype=np.float32)
        gt = None if geom_texture is None else np.ascontiguousarray(geom_texture, dtype=np.uint32)
        keep += [g, tc, gt]
        texs = [np.ascontiguousarray(t, dtype=np.uint8) for t in (textures or [])]
        tarr = (TextureDesc * max(1, len(texs)))()
        for k, t in enumerate(texs):
            assert t.ndim == 3 and t.shape[2] == 4, "textures are [H, W, 4] RGBA8"
            tarr[k] = TextureDesc(t.shape[1], t.shape[0], t.ctypes.data)
        desc = SceneDesc(v.shape[0], _ptr(v), _ptr(g), _ptr(tc),
                         0 if gt is None else gt.shape[0], _ptr(gt), len(texs),
                         C.cast(tarr, C.c_void_p) if texs else None, device)
        _check(lib().vsr_scene_create(C.byref(desc), C.byref(self._h)))
        del keep, texs

    @classmethod
    def from_workload(cls, scene, device: int = 0):
        return cls(scene.vertices, scene.geom_ids, scene.texcoords, scene.geom_texture,
                   scene.textures, device)

    # -- lifecycle ------------------------------------------------------------
    def close(self):
        if self._h:
            lib().vsr_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- setup ----------------------------------------------------------------
    def build(self, max_leaf_size=2, sah_bins=16, traversal_cost=1.0, intersection_cost=1.0):
        prm = BuildParams(max_leaf_size, sah_bins, traversal_cost, intersection_cost)
        _check(lib().vsr_bvh_build(self._h, C.byref(prm)))
        return self

    def build_gpu(self, max_leaf_size=2):
        """vsr_bvh_build_gpu: linear BVH built on the scene's GPU (NEXT-3)."""
        _check(lib().vsr_bvh_build_gpu(self._h, max_leaf_size))
        return self

    def build_ploc(self, max_leaf_size=2, radius=16):
        """vsr_bvh_build_ploc: GPU build by PLOC clustering (NEXT-3)."""
        _check(lib().vsr_bvh_build_ploc(self._h, max_leaf_size, radius))
        return self

    def build_wide(self):
        """vsr_bvh8_build: collapse the built binary BVH into the 8-wide compressed BVH."""
        _check(lib().vsr_bvh8_build(self._h))
        return self

    def trace_wide(self, rays, query=CLOSEST, isect=DEFAULT, hits=None, counts=None, stream=None,
                   alpha_threshold=0.01, checker_freq=8):
        """vsr_trace_bvh8 on device tensors (after build_wide); returns (hits, counts)."""
        import torch
        n = rays.shape[0]
        _check_rays(rays, n, self.device)
        if hits is None:
            hits = torch.empty((n, 4), dtype=torch.float32, device=rays.device)
        if isect in (COUNT, COUNT_ALPHA_TEXTURE) and counts is None:
            counts = torch.empty((n, 4), dtype=torch.int32, device=rays.device)
        _check_dev(hits, "hits", _f32(), n, (4,), self.device)
        _check_dev(counts, "counts", _i32(), n, (4,), self.device, optional=True)
        prm = IsectParams(alpha_threshold, checker_freq)
        _check(lib().vsr_trace_bvh8(self._h, _ptr(rays), n, query, isect, C.byref(prm), _ptr(hits),
                                    _ptr(counts), _stream_handle(stream, self.device)))
        return hits, counts

    def export_wide(self) -> dict:
        """Host copies of the 8-wide BVH: nodes [num_nodes, 20] uint32 (80-B WideNode),
        tris [num_tris, 12] uint32, sides [num_tris, 8] uint32 (wide leaf order)."""
        v = Bvh8View()
        _check(lib().vsr_bvh8_export(self._h, C.byref(v)))
        arrs = {"nodes": np.zeros((v.num_nodes, 20), np.uint32),
                "tris": np.zeros((v.num_tris, 12), np.uint32),
                "sides": np.zeros((v.num_tris, 8), np.uint32)}
        v.nodes, v.tris, v.sides = _ptr(arrs["nodes"]), _ptr(arrs["tris"]), _ptr(arrs["sides"])
        _check(lib().vsr_bvh8_export(self._h, C.byref(v)))
        arrs.update(root_lo=np.array(v.root_lo, np.float32), root_hi=np.array(v.root_hi, np.float32),
                    max_depth=int(v.max_depth), build_ms=float(v.build_ms))
        return arrs

    def stats(self) -> dict:
        s = Stats()
        _check(lib().vsr_scene_stats(self._h, C.byref(s)))
        return s.as_dict()

    # -- hot path ---------------------------------------------------------------
    def trace(self, rays, query=CLOSEST, isect=DEFAULT, hits=None, counts=None, stream=None,
              alpha_threshold=0.01, checker_freq=8, n=None):
        """Enqueue vsr_trace on device tensors; returns (hits, counts) tensors.

        rays: torch float32 CUDA tensor [n, 8]; hits: [n, 4] float32 (allocated if None);
        counts: [n, 4] int32 for COUNT kinds (allocated if None)."""
        import torch
        n = rays.shape[0] if n is None else n
        _check_rays(rays, n, self.device)
        if hits is None:
            hits = torch.empty((n, 4), dtype=torch.float32, device=rays.device)
        if isect in (COUNT, COUNT_ALPHA_TEXTURE) and counts is None:
            counts = torch.empty((n, 4), dtype=torch.int32, device=rays.device)
        _check_dev(hits, "hits", _f32(), n, (4,), self.device)
        _check_dev(counts, "counts", _i32(), n, (4,), self.device, optional=True)
        prm = IsectParams(alpha_threshold, checker_freq)
        _check(lib().vsr_trace(self._h, _ptr(rays), n, query, isect, C.byref(prm), _ptr(hits),
                               _ptr(counts), _stream_handle(stream, self.device)))
        return hits, counts

    def trace_pinhole(self, camera, query=CLOSEST, isect=DEFAULT, hits=None, counts=None,
                      stream=None, alpha_threshold=0.01, checker_freq=8):
        """vsr_trace_pinhole: primary rays generated in the kernel from `camera`
        (pinhole_camera(...)); returns (hits [n, 4], counts or None) in ray order."""
        import torch
        n = camera.width * camera.height * camera.spp
        if hits is None:
            hits = torch.empty((n, 4), dtype=torch.float32, device=f"cuda:{self.device}")
        if isect in (COUNT, COUNT_ALPHA_TEXTURE) and counts is None:
            counts = torch.empty((n, 4), dtype=torch.int32, device=hits.device)
        _check_dev(hits, "hits", _f32(), n, (4,), self.device)
        _check_dev(counts, "counts", _i32(), n, (4,), self.device, optional=True)
        prm = IsectParams(alpha_threshold, checker_freq)
        _check(lib().vsr_trace_pinhole(self._h, C.byref(camera), query, isect, C.byref(prm),
                                       _ptr(hits), _ptr(counts),
                                       _stream_handle(stream, self.device)))
        return hits, counts

    def trace_tiles(self, rays, tile_rays, rank, world, frame_hits_ptr, query=CLOSEST,
                    isect=DEFAULT, frame_counts_ptr=None, stream=None, alpha_threshold=0.01,
                    checker_freq=8):
        """vsr_trace_tiles: trace this rank's tile shard `rays` and store each hit at its frame
        position in the buffer at `frame_hits_ptr` (e.g. rank 0's frame via ipc_open)."""
        _check_rays(rays, rays.shape[0], self.device)
        prm = IsectParams(alpha_threshold, checker_freq)
        _check(lib().vsr_trace_tiles(self._h, _ptr(rays), rays.shape[0], tile_rays, rank, world,
                                     query, isect, C.byref(prm), frame_hits_ptr,
                                     frame_counts_ptr, _stream_handle(stream, self.device)))

    def trace_primitives(self, rays, query=CLOSEST, isect=DEFAULT, stream=None,
                         alpha_threshold=0.01, checker_freq=8):
        """vsr_trace_primitives: the query on the triangles as a plain list (no BVH)."""
        import torch
        n = rays.shape[0]
        _check_rays(rays, n, self.device)
        hits = torch.empty((n, 4), dtype=torch.float32, device=rays.device)
        counts = (torch.empty((n, 4), dtype=torch.int32, device=rays.device)
                  if isect in (COUNT, COUNT_ALPHA_TEXTURE) else None)
        prm = IsectParams(alpha_threshold, checker_freq)
        _check(lib().vsr_trace_primitives(self._h, _ptr(rays), n, query, isect, C.byref(prm),
                                          _ptr(hits), _ptr(counts),
                                          _stream_handle(stream, self.device)))
        return hits, counts

    def trace_multi(self, rays, max_hits, isect=DEFAULT, hits=None, num_hits=None, counts=None,
                    stream=None, alpha_threshold=0.01, checker_freq=8):
        """vsr_trace_multi: the max_hits smallest-t accepted hits per ray, ascending.

        Returns (hits [n, max_hits, 4] float32, num_hits [n] int32, counts or None)."""
        import torch
        n = rays.shape[0]
        _check_rays(rays, n, self.device)
        if hits is None:
            hits = torch.empty((n, max_hits, 4), dtype=torch.float32, device=rays.device)
        if num_hits is None:
            num_hits = torch.empty((n,), dtype=torch.int32, device=rays.device)
        if isect in (COUNT, COUNT_ALPHA_TEXTURE) and counts is None:
            counts = torch.empty((n, 4), dtype=torch.int32, device=rays.device)
        _check_dev(hits, "hits", _f32(), n, (max_hits, 4), self.device)
        _check_dev(num_hits, "num_hits", _i32(), n, (), self.device)
        _check_dev(counts, "counts", _i32(), n, (4,), self.device, optional=True)
        prm = IsectParams(alpha_threshold, checker_freq)
        _check(lib().vsr_trace_multi(self._h, _ptr(rays), n, max_hits, isect, C.byref(prm),
                                     _ptr(hits), _ptr(num_hits), _ptr(counts),
                                     _stream_handle(stream, self.device)))
        return hits, num_hits, counts

    def trace_raw(self, rays_ptr, n, query, isect, hits_ptr, counts_ptr=None, stream=0,
                  alpha_threshold=0.01, checker_freq=8):
        prm = IsectParams(alpha_threshold, checker_freq)
        _check(lib().vsr_trace(self._h, rays_ptr, n, query, isect, C.byref(prm), hits_ptr,
                               counts_ptr, stream))

    def trace_host(self, rays, query=CLOSEST, isect=DEFAULT, hits=None, counts=None, stream=None,
                   alpha_threshold=0.01, checker_freq=8):
        """vsr_trace_host over host buffers (numpy arrays or pinned CPU tensors)."""
        n = rays.shape[0]
        if hits is None:
            hits = np.empty(n, dtype=HIT_DTYPE)
        if isect in (COUNT, COUNT_ALPHA_TEXTURE) and counts is None:
            counts = np.empty(n, dtype=COUNTS_DTYPE)
        _check_host(rays, "rays", n, 32)
        _check_host(hits, "hits", n, 16)
        if counts is not None:
            _check_host(counts, "counts", n, 16)
        prm = IsectParams(alpha_threshold, checker_freq)
        _check(lib().vsr_trace_host(self._h, _ptr(rays), n, query, isect, C.byref(prm),
                                    _ptr(hits), _ptr(counts),
                                    0 if stream is None else _stream_handle(stream)))
        return hits, counts

    # -- replication (multi-GPU) ------------------------------------------------
    def export(self) -> dict:
        """Host copies of the flattened structure in the export layout."""
        v = BvhView()
        _check(lib().vsr_bvh_export(self._h, C.byref(v)))
        arrs = {
            "nodes": np.zeros((v.num_nodes, 16), np.uint32),
            "tris": np.zeros((v.num_tris, 12), np.uint32),
            "sides": np.zeros((v.num_tris, 8), np.uint32),
            "texdescs": np.zeros((v.num_textures, 4), np.uint32),
            "texels": np.zeros(v.num_texels, np.uint8),   # alpha plane (A8)
        }
        v.nodes, v.tris, v.sides, v.texdescs, v.texels = (
            _ptr(arrs["nodes"]) if v.num_nodes else None, _ptr(arrs["tris"]), _ptr(arrs["sides"]),
            _ptr(arrs["texdescs"]), _ptr(arrs["texels"]))
        _check(lib().vsr_bvh_export(self._h, C.byref(v)))
        arrs["root_ref"] = int(v.root_ref)
        arrs["root_lo"] = np.array(v.root_lo, np.float32)
        arrs["root_hi"] = np.array(v.root_hi, np.float32)
        return arrs

    @classmethod
    def import_arrays(cls, arrs: dict, device: int = 0):
        """vsr_scene_import from host numpy arrays or device tensors (export layout)."""
        v = BvhView()
        v.root_ref = int(arrs["root_ref"])
        v.root_lo = (C.c_float * 3)(*[float(x) for x in arrs["root_lo"]])
        v.root_hi = (C.c_float * 3)(*[float(x) for x in arrs["root_hi"]])
        v.num_nodes = arrs["nodes"].shape[0]
        v.num_tris = arrs["tris"].shape[0]
        v.num_textures = arrs["texdescs"].shape[0]
        v.num_texels = arrs["texels"].shape[0]
        v.nodes = _ptr(arrs["nodes"]) if v.num_nodes else None
        v.tris = _ptr(arrs["tris"])
        v.sides = _ptr(arrs["sides"])
        v.texdescs = _ptr(arrs["texdescs"])
        v.texels = _ptr(arrs["texels"])
        h = C.c_void_p()
        _check(lib().vsr_scene_import(C.byref(v), device, C.byref(h)))
        return cls(device=device, _handle=h)


class Group:
    """A list of built scenes queried as one (vsr_group_create / vsr_trace_group)."""

    def __init__(self, scenes):
        self.scenes = list(scenes)   # keep the scenes alive while the group exists
        arr = (C.c_void_p * len(self.scenes))(*[s._h.value for s in self.scenes])
        self._h = C.c_void_p()
        _check(lib().vsr_group_create(C.cast(arr, C.c_void_p), len(self.scenes),
                                      C.byref(self._h)))

    def close(self):
        if self._h:
            lib().vsr_group_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def trace(self, rays, query=CLOSEST, isect=DEFAULT, hits=None, which=None, counts=None,
              stream=None, alpha_threshold=0.01, checker_freq=8):
        """Returns (hits [n, 4], which [n] int32 list index, counts or None)."""
        import torch
        n = rays.shape[0]
        dev = self.scenes[0].device if self.scenes else None
        _check_rays(rays, n, dev)
        if hits is None:
            hits = torch.empty((n, 4), dtype=torch.float32, device=rays.device)
        if which is None:
            which = torch.empty((n,), dtype=torch.int32, device=rays.device)
        if isect in (COUNT, COUNT_ALPHA_TEXTURE) and counts is None:
            counts = torch.empty((n, 4), dtype=torch.int32, device=rays.device)
        _check_dev(hits, "hits", _f32(), n, (4,), dev)
        _check_dev(which, "which", _i32(), n, (), dev)
        _check_dev(counts, "counts", _i32(), n, (4,), dev, optional=True)
        prm = IsectParams(alpha_threshold, checker_freq)
        _check(lib().vsr_trace_group(self._h, _ptr(rays), n, query, isect, C.byref(prm),
                                     _ptr(hits), _ptr(which), _ptr(counts),
                                     _stream_handle(stream, dev)))
        return hits, which, counts

    def trace_multi(self, rays, max_hits, isect=DEFAULT, stream=None, alpha_threshold=0.01,
                    checker_freq=8):
        """vsr_trace_group_multi: (hits [n, k, 4], num_hits [n], which [n, k], counts or None)."""
        return _compound_multi(lib().vsr_trace_group_multi, self._h, rays, max_hits, isect,
                               stream, alpha_threshold, checker_freq,
                               self.scenes[0].device if self.scenes else None)


def _compound_multi(fn, handle, rays, max_hits, isect, stream, alpha_threshold, checker_freq,
                    device=None):
    import torch
    n = rays.shape[0]
    _check_rays(rays, n, device)
    hits = torch.empty((n, max_hits, 4), dtype=torch.float32, device=rays.device)
    num = torch.empty((n,), dtype=torch.int32, device=rays.device)
    which = torch.empty((n, max_hits), dtype=torch.int32, device=rays.device)
    counts = (torch.empty((n, 4), dtype=torch.int32, device=rays.device)
              if isect in (COUNT, COUNT_ALPHA_TEXTURE) else None)
    prm = IsectParams(alpha_threshold, checker_freq)
    _check(fn(handle, _ptr(rays), n, max_hits, isect, C.byref(prm), _ptr(hits), _ptr(num),
              _ptr(which), _ptr(counts), _stream_handle(stream, device)))
    return hits, num, which, counts


class Instances:
    """Two-level instancing (vsr_instances_create / vsr_trace_instances): a top-level BVH
    over instances of built scenes, each seen through an object_from_world [A | b] map."""

    def __init__(self, scenes, bvh, object_from_world, max_leaf_size=1, sah_bins=16):
        self.scenes = list(scenes)   # keep the scenes alive while the instances exist
        bvh = np.ascontiguousarray(bvh, dtype=np.uint32).reshape(-1)
        m = np.ascontiguousarray(object_from_world, dtype=np.float32).reshape(-1, 12)
        assert m.shape[0] == bvh.shape[0], "one 3x4 matrix per instance"
        arr = (Instance * max(1, bvh.shape[0]))()
        for k in range(bvh.shape[0]):
            arr[k].bvh = int(bvh[k])
            arr[k].object_from_world = (C.c_float * 12)(*m[k].tolist())
        sc = (C.c_void_p * len(self.scenes))(*[s._h.value for s in self.scenes])
        prm = BuildParams(max_leaf_size, sah_bins, 1.0, 1.0)
        self._h = C.c_void_p()
        _check(lib().vsr_instances_create(C.cast(sc, C.c_void_p), len(self.scenes),
                                          C.cast(arr, C.c_void_p), bvh.shape[0], C.byref(prm),
                                          C.byref(self._h)))

    def close(self):
        if self._h:
            lib().vsr_instances_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def trace(self, rays, query=CLOSEST, isect=DEFAULT, hits=None, inst=None, counts=None,
              stream=None, alpha_threshold=0.01, checker_freq=8):
        """Returns (hits [n, 4], inst [n] int32 caller instance index, counts or None)."""
        import torch
        n = rays.shape[0]
        dev = self.scenes[0].device if self.scenes else None
        _check_rays(rays, n, dev)
        if hits is None:
            hits = torch.empty((n, 4), dtype=torch.float32, device=rays.device)
        if inst is None:
            inst = torch.empty((n,), dtype=torch.int32, device=rays.device)
        if isect in (COUNT, COUNT_ALPHA_TEXTURE) and counts is None:
            counts = torch.empty((n, 4), dtype=torch.int32, device=rays.device)
        _check_dev(hits, "hits", _f32(), n, (4,), dev)
        _check_dev(inst, "inst", _i32(), n, (), dev)
        _check_dev(counts, "counts", _i32(), n, (4,), dev, optional=True)
        prm = IsectParams(alpha_threshold, checker_freq)
        _check(lib().vsr_trace_instances(self._h, _ptr(rays), n, query, isect, C.byref(prm),
                                         _ptr(hits), _ptr(inst), _ptr(counts),
                                         _stream_handle(stream, dev)))
        return hits, inst, counts

    def trace_multi(self, rays, max_hits, isect=DEFAULT, stream=None, alpha_threshold=0.01,
                    checker_freq=8):
        """vsr_trace_instances_multi: (hits [n, k, 4], num_hits [n], inst [n, k], counts)."""
        return _compound_multi(lib().vsr_trace_instances_multi, self._h, rays, max_hits, isect,
                               stream, alpha_threshold, checker_freq,
                               self.scenes[0].device if self.scenes else None)

    def export(self) -> dict:
        """Host copies of the top level: nodes [num_nodes, 16] uint32 (pair nodes) and
        records [num_instances, 16] uint32 (12 matrix floats, bvh, index, pad, pad)."""
        v = InstancesView()
        _check(lib().vsr_instances_export(self._h, C.byref(v)))
        nodes = np.zeros((v.num_nodes, 16), np.uint32)
        recs = np.zeros((v.num_instances, 16), np.uint32)
        v.nodes = _ptr(nodes) if v.num_nodes else None
        v.records = _ptr(recs)
        _check(lib().vsr_instances_export(self._h, C.byref(v)))
        return {"root_ref": int(v.root_ref), "root_lo": np.array(v.root_lo, np.float32),
                "root_hi": np.array(v.root_hi, np.float32), "nodes": nodes, "records": recs,
                "max_depth": int(v.max_depth), "r_safe": float(v.r_safe)}


# ---- device buffers shared across processes (CUDA IPC) ----------------------------------
def device_alloc(nbytes: int, device: int) -> int:
    p = C.c_void_p()
    _check(lib().vsr_device_alloc(nbytes, device, C.byref(p)))
    return p.value


def device_free(ptr: int, device: int):
    _check(lib().vsr_device_free(ptr, device))


def ipc_handle(ptr: int) -> bytes:
    h = (C.c_uint8 * 64)()
    _check(lib().vsr_ipc_handle(ptr, h))
    return bytes(h)


def ipc_open(handle: bytes, device: int) -> int:
    h = (C.c_uint8 * 64)(*handle)
    p = C.c_void_p()
    _check(lib().vsr_ipc_open(h, device, C.byref(p)))
    return p.value


def ipc_close(ptr: int, device: int):
    _check(lib().vsr_ipc_close(ptr, device))


class DeviceArray:
    """A raw device pointer seen by torch without a copy (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def hits_to_numpy(hits) -> np.ndarray:
    """[n,4] float32 tensor/array -> structured HIT_DTYPE array (prim as uint32 bits)."""
    if hasattr(hits, "detach"):
        hits = hits.detach().cpu().numpy()
    return np.ascontiguousarray(hits, dtype=np.float32).view(HIT_DTYPE).reshape(-1)


def counts_to_numpy(counts) -> np.ndarray:
    if hasattr(counts, "detach"):
        counts = counts.detach().cpu().numpy()
    return np.ascontiguousarray(counts).view(np.uint32).view(COUNTS_DTYPE).reshape(-1)
