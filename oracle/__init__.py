"""oracle — TEST INFRASTRUCTURE ONLY.

Plain CPU oracle for the custom-intersector hot path of arXiv 1912.12786
(oracle S: brute force, oracle.c; oracle BVH + contract walker C, walker.c).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_1912_12786_b200``) never imports it and it never imports
the product; the two share no code.  See oracle/oracle.h for citations.

Parity status (DESIGN.md §"Oracle pins"): every function here is pinned by
``tests/test_oracle_pins.py`` (closed forms, brute force, invariants); none
is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")

CLOSEST, ANY = 0, 1
NONE, DEFAULT, ALPHA_TEX, ALPHA_PROC, COUNT = 0, 1, 2, 3, 4
ALPHA_TEX_BILINEAR, ALPHA_PROC_UV = 5, 6     # NEXT-4 sampling variants (reading A28)
X1, X2, X3, X4, X5 = 1, 2, 4, 8, 16

HIT_DTYPE = np.dtype([("t", "<f4"), ("u", "<f4"), ("v", "<f4"), ("prim", "<u4")])
COUNT_DTYPE = np.dtype([("boxes", "<u4"), ("tris", "<u4"), ("alpha", "<u4")])


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, IEEE semantics)."""
    srcs = [os.path.join(_HERE, f) for f in ("oracle.c", "walker.c")]
    hdr = os.path.join(_HERE, "oracle.h")
    if not force and os.path.exists(LIB_PATH):
        newest = max(os.path.getmtime(p) for p in srcs + [hdr])
        if os.path.getmtime(LIB_PATH) >= newest:
            return LIB_PATH
    cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
           "-fno-strict-aliasing", "-pthread", "-D_GNU_SOURCE", "-Wall", "-Wno-unused-function",
           "-o", LIB_PATH + ".tmp"] + srcs + ["-lm"]
    subprocess.check_call(cmd)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


class _Scene(C.Structure):
    _fields_ = [("num_tris", C.c_uint32), ("vertices", C.c_void_p), ("geom_ids", C.c_void_p),
                ("texcoords", C.c_void_p), ("num_geoms", C.c_uint32),
                ("geom_texture", C.c_void_p), ("num_textures", C.c_uint32),
                ("tex_w", C.c_void_p), ("tex_h", C.c_void_p), ("tex_rgba", C.c_void_p)]


class _Hit(C.Structure):
    _fields_ = [("t", C.c_float), ("u", C.c_float), ("v", C.c_float), ("prim", C.c_uint32)]


class _Bvh(C.Structure):
    _fields_ = [("root_ref", C.c_uint32), ("root_lo", C.c_float * 3), ("root_hi", C.c_float * 3),
                ("num_nodes", C.c_uint32), ("num_tris", C.c_uint32), ("num_textures", C.c_uint32),
                ("nodes", C.c_void_p), ("tris", C.c_void_p), ("sides", C.c_void_p),
                ("texdescs", C.c_void_p), ("texels", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        mutant = os.environ.get("ORACLE_MUTANT_LIB")   # tools/mutate_oracle.py only
        if mutant:
            L = C.CDLL(mutant)
        else:
            build()
            L = C.CDLL(LIB_PATH)
        L.oracle_trace.argtypes = [C.POINTER(_Scene), C.c_void_p, C.c_uint64, C.c_int, C.c_int,
                                   C.c_float, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_int]
        L.oracle_eval_pair.argtypes = [C.POINTER(_Scene), C.c_void_p, C.c_uint32, C.c_int,
                                       C.c_float, C.c_uint32, C.POINTER(_Hit)]
        L.oracle_eval_pairs.argtypes = [C.POINTER(_Scene), C.c_void_p, C.c_void_p, C.c_uint64,
                                        C.c_int, C.c_float, C.c_uint32, C.c_void_p, C.c_void_p]
        L.walker_trace_wide.argtypes = [C.POINTER(_Bvh), C.c_void_p, C.c_uint32, C.c_void_p,
                                        C.c_uint64, C.c_int, C.c_int, C.c_float, C.c_uint32,
                                        C.c_void_p, C.c_void_p, C.c_int]
        L.oracle_mt.argtypes = [C.c_void_p] * 4 + [C.c_float] + [C.POINTER(C.c_float)] * 3
        L.oracle_tex_alpha.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p, C.c_float, C.c_float]
        L.oracle_tex_alpha.restype = C.c_float
        L.oracle_tex_alpha_bilinear.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p, C.c_float,
                                                C.c_float]
        L.oracle_tex_alpha_bilinear.restype = C.c_float
        L.oracle_lerp2.argtypes = [C.c_void_p] * 3 + [C.c_float, C.c_float, C.c_void_p]
        L.oracle_build_bvh.argtypes = [C.POINTER(_Scene), C.c_uint32, C.POINTER(_Bvh)]
        L.oracle_bvh_free.argtypes = [C.POINTER(_Bvh)]
        L.walker_trace.argtypes = [C.POINTER(_Bvh), C.c_void_p, C.c_uint64, C.c_int, C.c_int,
                                   C.c_float, C.c_uint32, C.c_void_p, C.c_void_p, C.c_int]
        L.walker_slab.argtypes = [C.c_void_p] * 3 + [C.c_float, C.POINTER(C.c_float),
                                                       C.POINTER(C.c_float)]
        L.oracle_trace_multi.argtypes = [C.POINTER(_Scene), C.c_void_p, C.c_uint64, C.c_uint32,
                                         C.c_int, C.c_float, C.c_uint32, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_int]
        L.walker_trace_multi.argtypes = [C.POINTER(_Bvh), C.c_void_p, C.c_uint64, C.c_uint32,
                                         C.c_int, C.c_float, C.c_uint32, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_int]
        L.walker_trace_list.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, C.c_int,
                                        C.c_int, C.c_float, C.c_uint32, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_int]
        L.walker_trace_instances.argtypes = [C.POINTER(_Bvh), C.c_void_p, C.c_void_p, C.c_uint32,
                                             C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_float,
                                             C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_float, C.c_int]
        L.oracle_ray_to_object.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.walker_trace_list_multi.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64,
                                              C.c_uint32, C.c_int, C.c_float, C.c_uint32,
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_int]
        L.walker_trace_instances_multi.argtypes = [C.POINTER(_Bvh), C.c_void_p, C.c_void_p,
                                                   C.c_uint32, C.c_void_p, C.c_uint64, C.c_int,
                                                   C.c_uint32, C.c_int, C.c_float, C.c_uint32,
                                                   C.c_void_p, C.c_void_p, C.c_void_p,
                                                   C.c_void_p, C.c_float, C.c_int]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


class OracleScene:
    """or_scene view over a workloads.Scene (keeps the numpy arrays alive)."""

    def __init__(self, scene):
        self.vertices = np.ascontiguousarray(scene.vertices, dtype=np.float32)
        self.geom_ids = np.ascontiguousarray(scene.geom_ids, dtype=np.uint32)
        self.texcoords = np.ascontiguousarray(scene.texcoords, dtype=np.float32)
        self.geom_texture = np.ascontiguousarray(scene.geom_texture, dtype=np.uint32)
        texs = list(scene.textures) if scene.textures else [np.full((1, 1, 4), 255, np.uint8)]
        self.textures = [np.ascontiguousarray(t, dtype=np.uint8) for t in texs]
        self.tex_w = np.array([t.shape[1] for t in self.textures], dtype=np.uint32)
        self.tex_h = np.array([t.shape[0] for t in self.textures], dtype=np.uint32)
        self._ptrs = (C.c_void_p * len(self.textures))(*[t.ctypes.data for t in self.textures])
        self.c = _Scene(self.vertices.shape[0], _ptr(self.vertices), _ptr(self.geom_ids),
                        _ptr(self.texcoords), self.geom_texture.shape[0], _ptr(self.geom_texture),
                        len(self.textures), _ptr(self.tex_w), _ptr(self.tex_h),
                        C.cast(self._ptrs, C.c_void_p))


def _as_scene(scene):
    return scene if isinstance(scene, OracleScene) else OracleScene(scene)


def _rays(rays):
    data = rays.data if hasattr(rays, "data") and not isinstance(rays, np.ndarray) else rays
    return np.ascontiguousarray(data, dtype=np.float32).reshape(-1, 8)


def trace(scene, rays, query=CLOSEST, isect=DEFAULT, alpha_threshold=0.01, checker_freq=8,
          flags=False, ties=False, nthreads=None):
    """Brute-force oracle S.  Returns hits (HIT_DTYPE) [, flags uint32] [, ntie uint32]."""
    sc = _as_scene(scene)
    r = _rays(rays)
    n = r.shape[0]
    hits = np.empty(n, dtype=HIT_DTYPE)
    fl = np.zeros(n, dtype=np.uint32) if flags else None
    nt = np.zeros(n, dtype=np.uint32) if ties else None
    rc = lib().oracle_trace(C.byref(sc.c), _ptr(r), n, query, isect, alpha_threshold,
                            checker_freq, _ptr(hits), _ptr(fl), _ptr(nt),
                            nthreads or default_threads())
    if rc != 0:
        raise ValueError(f"oracle_trace failed ({rc})")
    out = [hits]
    if flags:
        out.append(fl)
    if ties:
        out.append(nt)
    return out[0] if len(out) == 1 else tuple(out)


def trace_multi(scene, rays, k, isect=DEFAULT, alpha_threshold=0.01, checker_freq=8,
                nthreads=None):
    """Brute-force multi-hit: (hits [n, k] HIT_DTYPE, nhits uint32[n], ncut uint32[n])."""
    sc = _as_scene(scene)
    r = _rays(rays)
    n = r.shape[0]
    hits = np.empty((n, k), dtype=HIT_DTYPE)
    nh = np.zeros(n, dtype=np.uint32)
    nc = np.zeros(n, dtype=np.uint32)
    rc = lib().oracle_trace_multi(C.byref(sc.c), _ptr(r), n, k, isect, alpha_threshold,
                                  checker_freq, _ptr(hits), _ptr(nh), _ptr(nc),
                                  nthreads or default_threads())
    if rc != 0:
        raise ValueError(f"oracle_trace_multi failed ({rc})")
    return hits, nh, nc


def eval_pair(scene, ray, prim, isect=DEFAULT, alpha_threshold=0.01, checker_freq=8):
    """(accepted, t, u, v) of one ray against one caller-indexed triangle."""
    sc = _as_scene(scene)
    r = np.ascontiguousarray(ray, dtype=np.float32).reshape(8)
    h = _Hit()
    acc = lib().oracle_eval_pair(C.byref(sc.c), _ptr(r), int(prim), isect, alpha_threshold,
                                 checker_freq, C.byref(h))
    return bool(acc), h.t, h.u, h.v


def eval_pairs(scene, rays, prims, isect=DEFAULT, alpha_threshold=0.01, checker_freq=8):
    """eval_pair over arrays: (accepted bool[n], hits HIT_DTYPE[n]) of ray i against
    caller-indexed triangle prims[i]."""
    sc = _as_scene(scene)
    r = _rays(rays)
    p = np.ascontiguousarray(prims, dtype=np.uint32).reshape(-1)
    assert p.shape[0] == r.shape[0]
    acc = np.zeros(r.shape[0], np.uint8)
    hits = np.empty(r.shape[0], dtype=HIT_DTYPE)
    if lib().oracle_eval_pairs(C.byref(sc.c), _ptr(r), _ptr(p), r.shape[0], isect,
                               alpha_threshold, checker_freq, _ptr(acc), _ptr(hits)) != 0:
        raise ValueError("oracle_eval_pairs: prim out of range")
    return acc.astype(bool), hits


def mt(ray, v0, v1, v2, tmax=None):
    r = np.ascontiguousarray(ray, dtype=np.float32).reshape(8)
    a = [np.ascontiguousarray(x, dtype=np.float32).reshape(3) for x in (v0, v1, v2)]
    t, u, v = C.c_float(), C.c_float(), C.c_float()
    hit = lib().oracle_mt(_ptr(r), _ptr(a[0]), _ptr(a[1]), _ptr(a[2]),
                          float(r[7] if tmax is None else tmax), C.byref(t), C.byref(u), C.byref(v))
    return bool(hit), t.value, u.value, v.value


def tex_alpha(tex, s, t):
    tex = np.ascontiguousarray(tex, dtype=np.uint8)
    return lib().oracle_tex_alpha(tex.shape[1], tex.shape[0], _ptr(tex), s, t)


def tex_alpha_bilinear(tex, s, t):
    tex = np.ascontiguousarray(tex, dtype=np.uint8)
    return lib().oracle_tex_alpha_bilinear(tex.shape[1], tex.shape[0], _ptr(tex), s, t)


def slab(lo, hi, ray, best_t=None):
    """(hit, tnear, tfar) of the walker's slab test (App. A.2)."""
    r = np.ascontiguousarray(ray, dtype=np.float32).reshape(8)
    lo = np.ascontiguousarray(lo, dtype=np.float32).reshape(3)
    hi = np.ascontiguousarray(hi, dtype=np.float32).reshape(3)
    tn, tf = C.c_float(), C.c_float()
    hit = lib().walker_slab(_ptr(lo), _ptr(hi), _ptr(r), float(r[7] if best_t is None else best_t),
                            C.byref(tn), C.byref(tf))
    return bool(hit), tn.value, tf.value


def lerp2(a, b, c, u, v):
    arrs = [np.ascontiguousarray(x, dtype=np.float32).reshape(2) for x in (a, b, c)]
    out = np.zeros(2, dtype=np.float32)
    lib().oracle_lerp2(_ptr(arrs[0]), _ptr(arrs[1]), _ptr(arrs[2]), u, v, _ptr(out))
    return out


# ----------------------------------------------------------------------------
# BVH in the export layout (DESIGN.md §"Data layout")
# ----------------------------------------------------------------------------

@dataclass
class BvhArrays:
    root_ref: int
    root_lo: np.ndarray      # float32[3]
    root_hi: np.ndarray      # float32[3]
    nodes: np.ndarray        # uint32[num_nodes, 16]  (64 B pair nodes)
    tris: np.ndarray         # uint32[num_tris, 12]   (48 B)
    sides: np.ndarray        # uint32[num_tris, 8]    (32 B)
    texdescs: np.ndarray     # uint32[num_textures, 4] (16 B: offset lo/hi, w, h)
    texels: np.ndarray       # uint8[total texels]  (alpha plane)

    def c_struct(self):
        keep = [np.ascontiguousarray(x) for x in (self.nodes, self.tris, self.sides,
                                                   self.texdescs, self.texels)]
        self._keep = keep
        return _Bvh(self.root_ref, (C.c_float * 3)(*self.root_lo.tolist()),
                    (C.c_float * 3)(*self.root_hi.tolist()), keep[0].shape[0], keep[1].shape[0],
                    keep[3].shape[0], _ptr(keep[0]), _ptr(keep[1]), _ptr(keep[2]), _ptr(keep[3]),
                    _ptr(keep[4]))


def walk_wide(bvh: BvhArrays, wnodes, rays, query=CLOSEST, isect=DEFAULT, alpha_threshold=0.01,
              checker_freq=8, nthreads=None):
    """Walker C over an 8-wide compressed BVH: `wnodes` uint32 [N, 20]
    (80-B nodes), `bvh` carrying the root box and the WIDE-ordered tris / sides (+ texdescs /
    texels).  Returns (hits HIT_DTYPE, counts COUNT_DTYPE)."""
    r = _rays(rays)
    n = r.shape[0]
    w = np.ascontiguousarray(wnodes, dtype=np.uint32).reshape(-1, 20)
    hits = np.empty(n, dtype=HIT_DTYPE)
    counts = np.empty(n, dtype=COUNT_DTYPE)
    cb = bvh.c_struct()
    rc = lib().walker_trace_wide(C.byref(cb), _ptr(w), w.shape[0], _ptr(r), n, query, isect,
                                 alpha_threshold, checker_freq, _ptr(hits), _ptr(counts),
                                 nthreads or default_threads())
    if rc != 0:
        raise ValueError(f"walker_trace_wide failed ({rc})")
    return hits, counts


def build_bvh(scene, max_leaf: int = 4) -> BvhArrays:
    """Oracle-side object-median BVH in the export layout."""
    sc = _as_scene(scene)
    b = _Bvh()
    rc = lib().oracle_build_bvh(C.byref(sc.c), max_leaf, C.byref(b))
    if rc != 0:
        lib().oracle_bvh_free(C.byref(b))
        raise ValueError(f"oracle_build_bvh failed ({rc})")

    def grab(ptr, count, width):
        if count == 0:
            return np.zeros((0, width), dtype=np.uint32)
        arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint32)), shape=(count * width,))
        return arr.copy().reshape(count, width)

    total = 0
    td = grab(b.texdescs, b.num_textures, 4)
    for row in td:
        total = max(total, int(row[0]) + (int(row[1]) << 32) + int(row[2]) * int(row[3]))
    texels = (np.ctypeslib.as_array(C.cast(b.texels, C.POINTER(C.c_uint8)), shape=(total,)).copy()
              if total else np.zeros(0, np.uint8))
    out = BvhArrays(b.root_ref, np.array(b.root_lo, dtype=np.float32),
                    np.array(b.root_hi, dtype=np.float32), grab(b.nodes, b.num_nodes, 16),
                    grab(b.tris, b.num_tris, 12), grab(b.sides, b.num_tris, 8), td, texels)
    lib().oracle_bvh_free(C.byref(b))
    return out


def walk(bvh: BvhArrays, rays, query=CLOSEST, isect=DEFAULT, alpha_threshold=0.01,
         checker_freq=8, nthreads=None):
    """Contract walker C.  Returns (hits HIT_DTYPE, counts COUNT_DTYPE)."""
    r = _rays(rays)
    n = r.shape[0]
    hits = np.empty(n, dtype=HIT_DTYPE)
    counts = np.empty(n, dtype=COUNT_DTYPE)
    cb = bvh.c_struct()
    rc = lib().walker_trace(C.byref(cb), _ptr(r), n, query, isect, alpha_threshold, checker_freq,
                            _ptr(hits), _ptr(counts), nthreads or default_threads())
    if rc != 0:
        raise ValueError(f"walker_trace failed ({rc})")
    return hits, counts


def walk_list(bvhs, rays, query=CLOSEST, isect=DEFAULT, alpha_threshold=0.01, checker_freq=8,
              nthreads=None):
    """Contract walker C over a LIST of BVHs: (hits, which uint32[n], counts)."""
    r = _rays(rays)
    n = r.shape[0]
    hits = np.empty(n, dtype=HIT_DTYPE)
    which = np.empty(n, dtype=np.uint32)
    counts = np.empty(n, dtype=COUNT_DTYPE)
    arr = (_Bvh * len(bvhs))(*[b.c_struct() for b in bvhs])
    rc = lib().walker_trace_list(arr, len(bvhs), _ptr(r), n, query, isect, alpha_threshold,
                                 checker_freq, _ptr(hits), _ptr(which), _ptr(counts),
                                 nthreads or default_threads())
    if rc != 0:
        raise ValueError(f"walker_trace_list failed ({rc})")
    return hits, which, counts


def walk_multi(bvh: BvhArrays, rays, k, isect=DEFAULT, alpha_threshold=0.01, checker_freq=8,
               nthreads=None):
    """Contract walker C, multi-hit query: (hits [n, k], nhits, counts)."""
    r = _rays(rays)
    n = r.shape[0]
    hits = np.empty((n, k), dtype=HIT_DTYPE)
    nh = np.zeros(n, dtype=np.uint32)
    counts = np.empty(n, dtype=COUNT_DTYPE)
    cb = bvh.c_struct()
    rc = lib().walker_trace_multi(C.byref(cb), _ptr(r), n, k, isect, alpha_threshold, checker_freq,
                                  _ptr(hits), _ptr(nh), _ptr(counts), nthreads or default_threads())
    if rc != 0:
        raise ValueError(f"walker_trace_multi failed ({rc})")
    return hits, nh, counts


# ----------------------------------------------------------------------------
# Two-level instancing (reading A27)
# ----------------------------------------------------------------------------

def ray_to_object(m, ray):
    """walker.c's ray map of reading A27 for one ray (8 floats)."""
    mm = np.ascontiguousarray(m, dtype=np.float32).reshape(12)
    r = np.ascontiguousarray(ray, dtype=np.float32).reshape(8)
    out = np.zeros(8, dtype=np.float32)
    lib().oracle_ray_to_object(_ptr(mm), _ptr(r), _ptr(out))
    return out


def rays_to_object(rays, m):
    """Reading A27 written out in numpy fp32 (one IEEE op per step, no FMA):
    o'_i = ((A_i0*o_x + A_i1*o_y) + A_i2*o_z) + b_i,  d'_i = (A_i0*d_x + A_i1*d_y) + A_i2*d_z."""
    r = _rays(rays)
    A = np.ascontiguousarray(m, dtype=np.float32).reshape(3, 4)
    out = r.copy()
    o, d = r[:, 0:3], r[:, 4:7]
    for i in range(3):
        a0, a1, a2, b = (np.float32(A[i, j]) for j in range(4))
        out[:, i] = ((a0 * o[:, 0] + a1 * o[:, 1]) + a2 * o[:, 2]) + b
        out[:, 4 + i] = (a0 * d[:, 0] + a1 * d[:, 1]) + a2 * d[:, 2]
    return out


def trace_instances(scenes, bvh, mats, rays, query=CLOSEST, isect=DEFAULT, alpha_threshold=0.01,
                    checker_freq=8, nthreads=None):
    """Brute force over every instance: instance j shows scenes[bvh[j]]
    through the [A | b] map mats[j]; its candidates are oracle S on the mapped rays.
    CLOSEST: min t over all instances (equal t: the lower instance index); ANY: the lowest
    instance index with an accepted hit.  Returns (hits, inst uint32, flags uint32, ntie
    uint32): flags = the winner's X-flags, plus X1 when another instance's best t is within
    1e-5 relative of the winner's; ntie = instances whose best t equals the winner's."""
    r = _rays(rays)
    n = r.shape[0]
    bvh = np.asarray(bvh, dtype=np.int64).reshape(-1)
    mats = np.asarray(mats, dtype=np.float32).reshape(-1, 12)
    sc = [_as_scene(s) for s in scenes]
    best = np.empty(n, dtype=HIT_DTYPE)
    best["t"] = np.inf
    best["u"] = 0
    best["v"] = 0
    best["prim"] = 0xFFFFFFFF
    inst = np.full(n, 0xFFFFFFFF, dtype=np.uint32)
    flags = np.zeros(n, dtype=np.uint32)
    all_t = np.full((len(bvh), n), np.inf, dtype=np.float64)
    for j in range(len(bvh)):
        h, fl = trace(sc[bvh[j]], rays_to_object(r, mats[j]), query, isect, alpha_threshold,
                      checker_freq, flags=True, nthreads=nthreads)
        hit = h["prim"] != 0xFFFFFFFF
        all_t[j, hit] = h["t"][hit]
        if query == ANY:
            take = hit & (inst == 0xFFFFFFFF)
        else:
            take = hit & (h["t"] < best["t"])
        best[take] = h[take]
        inst[take] = j
        flags[take] = fl[take]
    won = inst != 0xFFFFFFFF
    ntie = np.zeros(n, dtype=np.uint32)
    if won.any():
        tw = best["t"].astype(np.float64)
        eq = all_t == tw[None, :]
        ntie = np.where(won, eq.sum(axis=0), 0).astype(np.uint32)
        with np.errstate(invalid="ignore"):   # inf - inf on rays no instance hits
            near = np.abs(all_t - tw[None, :]) <= 1e-5 * np.maximum(np.abs(tw[None, :]), 1e-30)
        others = near.sum(axis=0) > 1
        flags |= np.where(won & others, X1, 0).astype(np.uint32)
    return best, inst, flags, ntie


def walk_instances(top, records, bottoms, rays, query=CLOSEST, isect=DEFAULT, alpha_threshold=0.01,
                   checker_freq=8, nthreads=None):
    """Contract walker C over a two-level hierarchy.  top: dict with root_ref, root_lo,
    root_hi, nodes [m, 16] uint32 and optionally r_safe (the product's far-origin bound,
    reading A27; absent = infinity); records [k, 16] uint32 (64 B or_instance, leaf order);
    bottoms: list of BvhArrays.  Returns (hits, inst uint32, counts)."""
    r = _rays(rays)
    n = r.shape[0]
    recs = np.ascontiguousarray(records, dtype=np.uint32).reshape(-1, 16)
    nodes = np.ascontiguousarray(top["nodes"], dtype=np.uint32).reshape(-1, 16)
    tb = _Bvh(int(top["root_ref"]), (C.c_float * 3)(*[float(x) for x in top["root_lo"]]),
              (C.c_float * 3)(*[float(x) for x in top["root_hi"]]), nodes.shape[0], recs.shape[0],
              0, _ptr(nodes) if nodes.shape[0] else None, None, None, None, None)
    arr = (_Bvh * len(bottoms))(*[b.c_struct() for b in bottoms])
    hits = np.empty(n, dtype=HIT_DTYPE)
    inst = np.empty(n, dtype=np.uint32)
    counts = np.empty(n, dtype=COUNT_DTYPE)
    rc = lib().walker_trace_instances(C.byref(tb), _ptr(recs), arr, len(bottoms), _ptr(r), n,
                                      query, isect, alpha_threshold, checker_freq, _ptr(hits),
                                      _ptr(inst), _ptr(counts), float(top.get("r_safe", np.inf)),
                                      nthreads or default_threads())
    if rc != 0:
        raise ValueError(f"walker_trace_instances failed ({rc})")
    return hits, inst, counts


def walk_list_multi(bvhs, rays, k, isect=DEFAULT, alpha_threshold=0.01, checker_freq=8,
                    nthreads=None):
    """Walker C, multi-hit over a LIST of BVHs: (hits [n, k], nhits, which [n, k], counts)."""
    r = _rays(rays)
    n = r.shape[0]
    hits = np.empty((n, k), dtype=HIT_DTYPE)
    nh = np.zeros(n, dtype=np.uint32)
    which = np.empty((n, k), dtype=np.uint32)
    counts = np.empty(n, dtype=COUNT_DTYPE)
    arr = (_Bvh * len(bvhs))(*[b.c_struct() for b in bvhs])
    rc = lib().walker_trace_list_multi(arr, len(bvhs), _ptr(r), n, k, isect, alpha_threshold,
                                       checker_freq, _ptr(hits), _ptr(nh), _ptr(which),
                                       _ptr(counts), nthreads or default_threads())
    if rc != 0:
        raise ValueError(f"walker_trace_list_multi failed ({rc})")
    return hits, nh, which, counts


def walk_instances_multi(top, records, bottoms, rays, k, isect=DEFAULT, alpha_threshold=0.01,
                         checker_freq=8, nthreads=None):
    """Walker C, multi-hit over instances: (hits [n, k], nhits, inst [n, k], counts)."""
    r = _rays(rays)
    n = r.shape[0]
    recs = np.ascontiguousarray(records, dtype=np.uint32).reshape(-1, 16)
    nodes = np.ascontiguousarray(top["nodes"], dtype=np.uint32).reshape(-1, 16)
    tb = _Bvh(int(top["root_ref"]), (C.c_float * 3)(*[float(x) for x in top["root_lo"]]),
              (C.c_float * 3)(*[float(x) for x in top["root_hi"]]), nodes.shape[0], recs.shape[0],
              0, _ptr(nodes) if nodes.shape[0] else None, None, None, None, None)
    arr = (_Bvh * len(bottoms))(*[b.c_struct() for b in bottoms])
    hits = np.empty((n, k), dtype=HIT_DTYPE)
    nh = np.zeros(n, dtype=np.uint32)
    inst = np.empty((n, k), dtype=np.uint32)
    counts = np.empty(n, dtype=COUNT_DTYPE)
    rc = lib().walker_trace_instances_multi(C.byref(tb), _ptr(recs), arr, len(bottoms), _ptr(r), n,
                                            CLOSEST, k, isect, alpha_threshold, checker_freq,
                                            _ptr(hits), _ptr(nh), _ptr(inst), _ptr(counts),
                                            float(top.get("r_safe", np.inf)),
                                            nthreads or default_threads())
    if rc != 0:
        raise ValueError(f"walker_trace_instances_multi failed ({rc})")
    return hits, nh, inst, counts

