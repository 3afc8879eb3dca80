"""GPU BVH builders: linear BVH (vsr_bvh_build_gpu) and PLOC clustering
(vsr_bvh_build_ploc).  The exported tree is structurally valid (tests/bvh_check.py), walker C on
it equals the brute force, and the GPU trace on it is bit-exact vs walker C (hits and counts) and
equals the SAH tree's results."""
import numpy as np
import pytest

import workloads as W
from tests import bvh_check

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
MISS = 0xFFFFFFFF


@pytest.fixture(scope="module")
def V():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_12786_b200 import _build
    _build.build()
    from paper_1912_12786_b200 import vsr
    return vsr


def trace(V, scene, rays, q, k):
    r = torch.from_numpy(np.ascontiguousarray(rays, np.float32)).cuda()
    h, c = scene.trace(r, q, k)
    torch.cuda.synchronize()
    return V.hits_to_numpy(h), (V.counts_to_numpy(c) if c is not None else None)


def build(V, sc, how, max_leaf):
    s = V.Scene.from_workload(sc)
    return s.build_gpu(max_leaf) if how == "lbvh" else s.build_ploc(max_leaf, 8 if how == "ploc8" else 16)


@pytest.mark.parametrize("how", ["lbvh", "ploc", "ploc8"])
@pytest.mark.parametrize("max_leaf", [1, 2, 4, 32])
def test_lbvh_valid_and_exact(V, oracle_lib, max_leaf, how):
    o = oracle_lib
    sc = W.random_soup(5000, seed=70 + max_leaf, size=1.5)
    rays = W.random_rays(5001, seed=71).data
    g = build(V, sc, how, max_leaf)
    e = g.export()
    depth = bvh_check.validate(e, sc.vertices, max_leaf)
    st = g.stats()
    assert depth == st["max_depth"] and e["nodes"].shape[0] == st["num_nodes"]
    b = bvh_check.to_oracle(e)
    ref, nt = o.trace(sc, rays, o.CLOSEST, o.ALPHA_TEX, ties=True)
    for q, oq in ((V.CLOSEST, o.CLOSEST), (V.ANY, o.ANY)):
        for k, ok in ((V.COUNT, o.DEFAULT), (V.COUNT_ALPHA_TEXTURE, o.ALPHA_TEX),
                      (V.ALPHA_PROCEDURAL, o.ALPHA_PROC)):
            h, c = trace(V, g, rays, q, k)
            wh, wc = o.walk(b, rays, oq, ok)
            assert np.array_equal(h.view(np.uint32), wh.view(np.uint32))
            if c is not None:
                assert np.array_equal(c["boxes"], wc["boxes"]) and np.array_equal(c["tris"], wc["tris"])
    h, _ = trace(V, g, rays, V.CLOSEST, V.ALPHA_TEXTURE)
    hit = ref["prim"] != MISS
    assert np.array_equal(h["prim"] != MISS, hit) and np.array_equal(h["t"], ref["t"])
    ok = nt <= 1
    assert np.array_equal(h[ok], ref[ok])


@pytest.mark.parametrize("how", ["lbvh", "ploc"])
def test_lbvh_equals_sah_on_forest(V, how):
    sc, rays = W.config("C2", 480, 272)
    a = V.Scene.from_workload(sc).build()
    g = build(V, sc, how, 2)
    bvh_check.validate(g.export(), sc.vertices, 2)
    for q in (V.CLOSEST, V.ANY):
        ha, _ = trace(V, a, rays.data, q, V.ALPHA_TEXTURE)
        hg, _ = trace(V, g, rays.data, q, V.ALPHA_TEXTURE)
        assert np.array_equal(ha["prim"] != MISS, hg["prim"] != MISS)
        if q == V.CLOSEST:
            assert np.array_equal(ha["t"], hg["t"])


@pytest.mark.parametrize("how", ["lbvh", "ploc"])
def test_lbvh_edge_cases(V, oracle_lib, how):
    o = oracle_lib
    # one triangle; all-coincident centroids (equal Morton codes); degenerate triangles
    one = W.stacked_quads(1)
    one.vertices, one.geom_ids, one.texcoords = one.vertices[:1], one.geom_ids[:1], one.texcoords[:1]
    s1 = build(V, one, how, 2)
    e1 = s1.export()
    assert e1["nodes"].shape[0] == 0 and e1["root_ref"] & 0x80000000
    two = W.stacked_quads(1)     # two triangles, max_leaf 1: one inner node
    s1b = build(V, two, how, 1)
    bvh_check.validate(s1b.export(), two.vertices, 1)
    same = W.stacked_quads(64, z0=1.0, dz=0.0)     # 128 triangles, pairwise-equal centroids
    s2 = build(V, same, how, 1)
    bvh_check.validate(s2.export(), same.vertices, 1)
    assert s2.stats()["max_depth"] <= 64
    sc = W.random_soup(300, seed=72)
    v = sc.vertices.copy()
    v[5, 3:6] = v[5, 0:3]
    v[9, 6:9] = v[9, 0:3]
    d = build(V, W.Scene("d", v, sc.geom_ids, sc.texcoords, sc.geom_texture, sc.textures), how, 2)
    st = d.stats()
    assert st["num_degenerate"] == 2 and st["num_tris"] == 298
    prims = set(d.export()["tris"][:, 3].tolist())
    assert 5 not in prims and 9 not in prims
    rays = W.random_rays(2000, seed=73).data
    ref = o.trace(W.Scene("d", v, sc.geom_ids, sc.texcoords, sc.geom_texture, sc.textures), rays,
                  o.CLOSEST, o.DEFAULT)
    h, _ = trace(V, d, rays, V.CLOSEST, V.DEFAULT)
    assert np.array_equal(h["t"], ref["t"])
    with pytest.raises(V.VsrError):
        V.Scene.from_workload(sc).build_gpu(0)
    with pytest.raises(V.VsrError):
        V.Scene.from_workload(sc).build_ploc(2, 0)
    with pytest.raises(V.VsrError):
        V.Scene.from_workload(sc, device=-1).build_gpu(2)
