"""GPU parity of the multi-hit query
through vsr_trace_multi, against the brute-force oracle and the contract walker."""
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


def okind(V, o, k):
    return {V.NONE: o.NONE, V.DEFAULT: o.DEFAULT, V.ALPHA_TEXTURE: o.ALPHA_TEX,
            V.ALPHA_PROCEDURAL: o.ALPHA_PROC, V.COUNT: o.DEFAULT,
            V.COUNT_ALPHA_TEXTURE: o.ALPHA_TEX}[k]


def gpu_multi(V, s, rays_np, k, isect):
    r = torch.from_numpy(np.ascontiguousarray(rays_np, np.float32)).cuda()
    hits, nh, counts = s.trace_multi(r, k, isect)
    torch.cuda.synchronize()
    h = V.hits_to_numpy(hits.reshape(-1, 4)).reshape(-1, k)
    c = V.counts_to_numpy(counts) if counts is not None else None
    return h, nh.cpu().numpy().astype(np.uint32), c


def check_vs_oracle(o, sc, rays_np, k, ok, h, nh):
    ref, rn, rcut = o.trace_multi(sc, rays_np, k, isect=ok)
    assert np.array_equal(nh, rn)
    assert np.array_equal(h["t"], ref["t"])             # the k smallest t, bit-exact
    diff = np.nonzero(np.any(h["prim"] != ref["prim"], axis=1))[0]
    for r in diff:
        # only equal-t groups may be ordered/cut differently: every GPU entry must be an
        # accepted candidate with exactly that t, u, v
        for j in range(nh[r]):
            acc, t, u, v = o.eval_pair(sc, rays_np[r], int(h["prim"][r, j]), ok)
            assert acc and t == h["t"][r, j] and u == h["u"][r, j] and v == h["v"][r, j]
        assert len(set(h["prim"][r][:nh[r]])) == nh[r]    # no duplicates
    same = ~np.isin(np.arange(len(nh)), diff)
    assert np.array_equal(h["u"][same], ref["u"][same]) and np.array_equal(h["v"][same], ref["v"][same])
    return len(diff)


@pytest.mark.parametrize("k", [1, 3, 4, 5, 16])
def test_multi_soup_and_c1(V, oracle_lib, k):
    o = oracle_lib
    for sc, rays in ((W.random_soup(900, seed=70 + k, size=3.5), W.random_rays(3001, seed=71)),
                     W.config("C1")):
        s = V.Scene.from_workload(sc).build()
        for kind in (V.NONE, V.DEFAULT, V.ALPHA_TEXTURE, V.ALPHA_PROCEDURAL):
            h, nh, _ = gpu_multi(V, s, rays.data, k, kind)
            check_vs_oracle(o, sc, rays.data, k, okind(V, o, kind), h, nh)


@pytest.mark.parametrize("k", [2, 7])
def test_multi_counts_vs_walker(V, oracle_lib, k):
    o = oracle_lib
    sc = W.random_soup(1200, seed=80, size=3.0)
    rays = W.random_rays(6000, seed=81)
    s = V.Scene.from_workload(sc).build()
    b = bvh_check.to_oracle(s.export())
    for kind in (V.COUNT, V.COUNT_ALPHA_TEXTURE):
        h, nh, c = gpu_multi(V, s, rays.data, k, kind)
        wh, wn, wc = o.walk_multi(b, rays.data, k, isect=okind(V, o, kind))
        assert h.tobytes() == wh.tobytes() and np.array_equal(nh, wn)
        for f in ("boxes", "tris", "alpha"):
            assert np.array_equal(c[f], wc[f])


def test_multi_k1_is_closest(V):
    sc, rays = W.config("C1")
    s = V.Scene.from_workload(sc).build()
    r = torch.from_numpy(rays.data).cuda()
    for kind in (V.DEFAULT, V.ALPHA_TEXTURE):
        hc, _ = s.trace(r, V.CLOSEST, kind)
        hm, _, _ = s.trace_multi(r, 1, kind)
        torch.cuda.synchronize()
        assert hc.cpu().numpy().tobytes() == hm.cpu().numpy().tobytes()


def test_multi_c2_sampled(V, oracle_lib):
    o = oracle_lib
    sc, rays = W.config("C2")
    s = V.Scene.from_workload(sc).build()
    h, nh, _ = gpu_multi(V, s, rays.data, 4, V.ALPHA_TEXTURE)
    idx = np.sort(np.random.default_rng(90).choice(rays.n, 1500, replace=False))
    check_vs_oracle(o, sc, rays.data[idx], 4, o.ALPHA_TEX, h[idx], nh[idx])
    assert nh.mean() > 0.5


def test_multi_errors(V):
    sc = W.quad_pair_scene()
    s = V.Scene.from_workload(sc).build()
    r = torch.zeros((8, 8), device="cuda")
    for bad_k in (0, 17):
        with pytest.raises(V.VsrError) as e:
            s.trace_multi(r, bad_k, V.DEFAULT)
        assert e.value.status == V.ERR_INVALID_ARG
    with pytest.raises(V.VsrError) as e:
        s.trace_multi(r, 4, V.RUNTIME_SWITCH_DEFAULT)
    assert e.value.status == V.ERR_UNSUPPORTED
