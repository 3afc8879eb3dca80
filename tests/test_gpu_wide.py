"""GPU parity of the 8-wide compressed BVH:
vsr_trace_bvh8 against walker C's wide walk (hits AND counts bit-exact: the traversal order,
the decode and the slab are the documented contract) and against oracle S (brute force),
on ragged soups, C1 and the full C2 frame in the bench's launch configuration."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import compare

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def V():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_12786_b200 import _build
    _build.build()
    from paper_1912_12786_b200 import vsr
    return vsr


def _walk_arrays(s):
    w = s.export_wide()
    b = s.export()
    arr = oracle.BvhArrays(0, w["root_lo"], w["root_hi"], np.zeros((0, 16), np.uint32), w["tris"],
                           w["sides"], b["texdescs"], b["texels"])
    return w["nodes"], arr


def _trace(V, s, rays, q, k):
    d = torch.from_numpy(np.ascontiguousarray(rays)).cuda()
    hits, counts = s.trace_wide(d, q, k)
    torch.cuda.synchronize()
    return V.hits_to_numpy(hits), (V.counts_to_numpy(counts) if counts is not None else None)


KINDS = [("NONE", oracle.NONE), ("DEFAULT", oracle.DEFAULT), ("ALPHA_TEXTURE", oracle.ALPHA_TEX),
         ("ALPHA_PROCEDURAL", oracle.ALPHA_PROC), ("ALPHA_TEXTURE_BILINEAR", oracle.ALPHA_TEX_BILINEAR),
         ("ALPHA_PROCEDURAL_UV", oracle.ALPHA_PROC_UV), ("COUNT", oracle.DEFAULT),
         ("COUNT_ALPHA_TEXTURE", oracle.ALPHA_TEX)]


@pytest.mark.parametrize("max_leaf", [1, 2, 4])
def test_wide_vs_walker_and_brute_force_soups(V, oracle_lib, max_leaf):
    sc = W.random_soup(3000, seed=40 + max_leaf)
    rays = W.random_rays(5000, seed=40 + max_leaf).data      # 39 blocks + a ragged tail
    s = V.Scene.from_workload(sc).build(max_leaf_size=max_leaf).build_wide()
    nodes, arr = _walk_arrays(s)
    for q, oq in ((V.CLOSEST, oracle.CLOSEST), (V.ANY, oracle.ANY)):
        for name, ok in KINDS:
            k = getattr(V, name)
            h, c = _trace(V, s, rays, q, k)
            wh, wc = oracle.walk_wide(arr, nodes, rays, oq, ok)
            assert h.tobytes() == wh.tobytes(), (name, q)
            if c is not None:
                for f in ("boxes", "tris", "alpha"):
                    assert np.array_equal(c[f], wc[f]), (name, q, f)
            if name in ("DEFAULT", "ALPHA_TEXTURE", "ALPHA_PROCEDURAL"):
                ref, nt = oracle.trace(sc, rays, oq, ok, ties=True)
                compare(oracle, sc, rays, oq, ok, h, ref, nt)


def test_wide_c1(V, oracle_lib):
    sc, rays = W.config("C1")
    s = V.Scene.from_workload(sc).build(max_leaf_size=1).build_wide()
    for q, oq in ((V.CLOSEST, oracle.CLOSEST), (V.ANY, oracle.ANY)):
        for name, ok in KINDS[:4]:
            h, _ = _trace(V, s, rays.data, q, getattr(V, name))
            ref, nt = oracle.trace(sc, rays.data, oq, ok, ties=True)
            compare(oracle, sc, rays.data, oq, ok, h, ref, nt)


@pytest.fixture(scope="module")
def c2(V):
    sc, rays = W.config("C2")
    s = V.Scene.from_workload(sc).build().build_wide()
    return sc, rays, s


def test_wide_c2_full_frame_vs_walker(V, oracle_lib, c2):
    sc, rays, s = c2
    nodes, arr = _walk_arrays(s)
    for q, oq, name, ok in ((V.ANY, oracle.ANY, "ALPHA_TEXTURE", oracle.ALPHA_TEX),
                            (V.CLOSEST, oracle.CLOSEST, "COUNT_ALPHA_TEXTURE", oracle.ALPHA_TEX)):
        h, c = _trace(V, s, rays.data, q, getattr(V, name))
        wh, wc = oracle.walk_wide(arr, nodes, rays.data, oq, ok)
        assert h.tobytes() == wh.tobytes()
        if c is not None:
            for f in ("boxes", "tris", "alpha"):
                assert np.array_equal(c[f], wc[f])


def test_wide_c2_equals_binary_and_oracle(V, oracle_lib, c2):
    sc, rays, s = c2
    d = torch.from_numpy(rays.data).cuda()
    for q in (V.CLOSEST, V.ANY):
        hb, _ = s.trace(d, q, V.ALPHA_TEXTURE)
        hw, _ = s.trace_wide(d, q, V.ALPHA_TEXTURE)
        torch.cuda.synchronize()
        hb, hw = V.hits_to_numpy(hb), V.hits_to_numpy(hw)
        assert np.array_equal(hb["prim"] != 0xFFFFFFFF, hw["prim"] != 0xFFFFFFFF)
        if q == V.CLOSEST:   # same MT arithmetic: t bit-equal, prims equal up to exact t ties
            assert np.array_equal(hb["t"], hw["t"])
    idx = np.sort(np.random.default_rng(77).choice(rays.n, 65536, replace=False))
    sub = np.ascontiguousarray(rays.data[idx])
    osc = oracle.OracleScene(sc)
    for q, oq in ((V.CLOSEST, oracle.CLOSEST), (V.ANY, oracle.ANY)):
        hw, _ = s.trace_wide(d, q, V.ALPHA_TEXTURE)
        torch.cuda.synchronize()
        g = V.hits_to_numpy(hw)[idx]
        ref, nt = (oracle.trace(osc, sub, oq, oracle.ALPHA_TEX, ties=True) if oq == oracle.CLOSEST
                   else (oracle.trace(osc, sub, oq, oracle.ALPHA_TEX), None))
        compare(oracle, osc, sub, oq, oracle.ALPHA_TEX, g, ref, nt)


def test_wide_errors(V):
    sc = W.random_soup(100, seed=3)
    s = V.Scene.from_workload(sc).build()
    r = torch.zeros((4, 8), device="cuda")
    with pytest.raises(V.VsrError) as e:
        s.trace_wide(r)
    assert e.value.status == V.ERR_NOT_BUILT
    s.build_wide()
    with pytest.raises(V.VsrError) as e:
        s.trace_wide(r, V.CLOSEST, V.RUNTIME_SWITCH_DEFAULT)
    assert e.value.status == V.ERR_UNSUPPORTED
    s.build(max_leaf_size=2)     # a rebuild drops the wide BVH
    with pytest.raises(V.VsrError) as e:
        s.trace_wide(r)
    assert e.value.status == V.ERR_NOT_BUILT
