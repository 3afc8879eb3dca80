"""8-wide compressed BVH, CPU only: the product's
collapse on host-only scenes (device -1) checked structurally, and walker C's wide walk
(oracle/walker.c walker_trace_wide, written from the documented layout) pinned to the plain
definition (oracle S brute force) and to hand counts."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import compare

V = pytest.importorskip("paper_1912_12786_b200.vsr")


@pytest.fixture(scope="module", autouse=True)
def _lib(oracle_lib):
    return oracle_lib


def _host_scene(sc, max_leaf=2):
    s = V.Scene.from_workload(sc, device=-1).build(max_leaf_size=max_leaf)
    return s.build_wide()


def _wide_arrays(s):
    w = s.export_wide()
    b = s.export()
    arr = oracle.BvhArrays(0, w["root_lo"], w["root_hi"], np.zeros((0, 16), np.uint32), w["tris"],
                           w["sides"], b["texdescs"], b["texels"])
    return w, arr


def _decode(nodes):
    """Decoded child boxes [N, 8, 2, 3] (lo/hi) in float32: plane = fl((2^23 + q) s + pm),
    evaluated exactly in float64 then rounded once (the documented decode)."""
    raw = nodes.view(np.uint8).reshape(-1, 80)
    pm = nodes[:, 0:3].view(np.float32).astype(np.float64)
    e = raw[:, 12:15].astype(np.int64)
    scale = np.ldexp(1.0, e - 127)
    q = raw[:, 32:80].reshape(-1, 2, 3, 8).astype(np.float64)      # [N, lo/hi, axis, slot]
    planes = ((8388608.0 + q) * scale[:, None, :, None] + pm[:, None, :, None]).astype(np.float32)
    return planes.transpose(0, 3, 1, 2)                            # [N, slot, lo/hi, axis]


def _tri_bounds(tris):
    tf = tris.view(np.float32)
    v0, e1, e2 = tf[:, 0:3], tf[:, 4:7], tf[:, 8:11]
    pts = np.stack([v0, v0 + e1, v0 + e2])
    return pts.min(axis=0), pts.max(axis=0)


@pytest.mark.parametrize("max_leaf", [1, 2, 4])
def test_structure_and_conservative_boxes(max_leaf):
    sc = W.random_soup(600, seed=31)
    s = _host_scene(sc, max_leaf)
    w, _ = _wide_arrays(s)
    nodes = w["nodes"]
    raw = nodes.view(np.uint8).reshape(-1, 80)
    imask = raw[:, 15]
    child_base = nodes[:, 4]
    tri_base = nodes[:, 5]
    meta = raw[:, 24:32]
    boxes = _decode(nodes)
    tlo, thi = _tri_bounds(w["tris"])
    n = nodes.shape[0]
    seen_node = np.zeros(n, np.int64)
    seen_tri = np.zeros(w["tris"].shape[0], np.int64)
    seen_node[0] = 1

    def subtree_tris(i):
        out = []
        for sl in range(8):
            m = int(meta[i, sl])
            if m == 0xFF:
                continue
            if (imask[i] >> sl) & 1:
                assert m == 0x80
                rank = bin(int(imask[i]) & ((1 << sl) - 1)).count("1")
                out += subtree_tris(int(child_base[i]) + rank)
            else:
                assert m < 0x80 and (m >> 5) + 1 <= max(1, min(max_leaf, 4))
                out += list(range(int(tri_base[i]) + (m & 31), int(tri_base[i]) + (m & 31) + (m >> 5) + 1))
        return out

    for i in range(n):
        for sl in range(8):
            m = int(meta[i, sl])
            if m == 0xFF:
                continue
            lo, hi = boxes[i, sl, 0], boxes[i, sl, 1]
            assert np.all(lo <= hi)
            if (imask[i] >> sl) & 1:
                rank = bin(int(imask[i]) & ((1 << sl) - 1)).count("1")
                c = int(child_base[i]) + rank
                assert 0 < c < n
                seen_node[c] += 1
                idx = subtree_tris(c)
            else:
                idx = list(range(int(tri_base[i]) + (m & 31), int(tri_base[i]) + (m & 31) + (m >> 5) + 1))
                seen_tri[idx] += 1
            # the decoded (quantized) child box contains every triangle below it
            assert np.all(lo <= tlo[idx].min(axis=0)) and np.all(hi >= thi[idx].max(axis=0))
    assert np.all(seen_node == 1) and np.all(seen_tri == 1)
    prims = w["tris"][:, 3]
    assert np.array_equal(np.sort(prims), np.arange(sc.num_tris))   # every triangle, once
    assert w["max_depth"] <= 64


@pytest.mark.parametrize("isect", [oracle.DEFAULT, oracle.ALPHA_TEX, oracle.ALPHA_PROC,
                                   oracle.ALPHA_TEX_BILINEAR, oracle.ALPHA_PROC_UV])
@pytest.mark.parametrize("max_leaf", [1, 4])
def test_walk_wide_equals_brute_force(isect, max_leaf):
    sc = W.random_soup(400, seed=7)
    rays = W.random_rays(3000, seed=7).data
    s = _host_scene(sc, max_leaf)
    w, arr = _wide_arrays(s)
    for q in (oracle.CLOSEST, oracle.ANY):
        h, c = oracle.walk_wide(arr, w["nodes"], rays, q, isect)
        ref, nt = oracle.trace(sc, rays, q, isect, ties=True)
        compare(oracle, sc, rays, q, isect, h, ref, nt)
        assert np.all(c["boxes"] >= 1) and np.all(c["tris"] <= sc.num_tris)


def test_walk_wide_c1_closed_form():
    sc, rays = W.config("C1")
    s = _host_scene(sc, 1)
    w, arr = _wide_arrays(s)
    for isect in (oracle.DEFAULT, oracle.ALPHA_TEX):
        h, _ = oracle.walk_wide(arr, w["nodes"], rays.data, oracle.CLOSEST, isect)
        ref, nt = oracle.trace(sc, rays.data, oracle.CLOSEST, isect, ties=True)
        compare(oracle, sc, rays.data, oracle.CLOSEST, isect, h, ref, nt)


def test_hand_counts_single_wide_node():
    """Three separated triangles, max_leaf 1: the wide root holds 3 leaf children.  A ray
    through the root box that misses all three costs 1 (root) + 3 (valid children) box tests
    and no triangle test; a ray missing the root box costs (1, 0); a ray hitting one
    triangle's box tests exactly that triangle."""
    tris = np.array([[0, 0, 0, 1, 0, 0, 0, 1, 0],
                     [3, 0, 0, 4, 0, 0, 3, 1, 0],
                     [6, 0, 0, 7, 0, 0, 6, 1, 0]], np.float32)
    sc = W.Scene("three", tris, np.zeros(3, np.uint32), np.zeros((3, 6), np.float32),
                 np.zeros(1, np.uint32), [np.full((1, 1, 4), 255, np.uint8)])
    s = _host_scene(sc, 1)
    w, arr = _wide_arrays(s)
    assert w["nodes"].shape[0] == 1
    rays = np.array([[2.0, 0.5, -1, 1e-4, 0, 0, 1, np.inf],      # between triangles 0 and 1
                     [2.0, 5.0, -1, 1e-4, 0, 0, 1, np.inf],      # misses the root box
                     [3.2, 0.3, -1, 1e-4, 0, 0, 1, np.inf]], np.float32)
    h, c = oracle.walk_wide(arr, w["nodes"], rays, oracle.CLOSEST, oracle.DEFAULT)
    assert (c["boxes"][0], c["tris"][0]) == (4, 0)
    assert (c["boxes"][1], c["tris"][1]) == (1, 0)
    assert (c["boxes"][2], c["tris"][2]) == (4, 1) and h["prim"][2] == 1 and h["t"][2] == 1.0


def test_wide_build_errors():
    sc = W.random_soup(50, seed=2)
    s = V.Scene.from_workload(sc, device=-1).build(max_leaf_size=8)
    with pytest.raises(V.VsrError) as e:
        s.build_wide()
    assert e.value.status == V.ERR_UNSUPPORTED
    s2 = V.Scene.from_workload(sc, device=-1)
    with pytest.raises(V.VsrError) as e:
        s2.build_wide()
    assert e.value.status == V.ERR_NOT_BUILT
