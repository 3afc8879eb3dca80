"""GPU parity of list-of-BVHs queries
through vsr_trace_group: hits vs brute force over the concatenated triangles,
counts and `which` bit-exact vs the list walker on the exported BVHs."""
import numpy as np
import pytest

import workloads as W
from tests import bvh_check
from tests.parity import compare

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


def run(V, g, rays_np, q, k):
    r = torch.from_numpy(np.ascontiguousarray(rays_np, np.float32)).cuda()
    hits, which, counts = g.trace(r, q, k)
    torch.cuda.synchronize()
    return (V.hits_to_numpy(hits), which.cpu().numpy().astype(np.uint32),
            V.counts_to_numpy(counts) if counts is not None else None)


@pytest.mark.parametrize("parts", [1, 3, 8])
def test_group_vs_bruteforce_and_walker(V, oracle_lib, parts):
    o = oracle_lib
    sc = W.random_soup(1500, seed=40 + parts, size=3.0)
    rays = W.random_rays(4001, seed=41)
    subs = W.split_scene(sc, parts)
    scenes = [V.Scene.from_workload(s).build() for s in subs]
    g = V.Group(scenes)
    cat, offs = W.concat_scenes(subs)
    bs = [bvh_check.to_oracle(s.export()) for s in scenes]
    for q, oq in ((V.CLOSEST, o.CLOSEST), (V.ANY, o.ANY)):
        for k in (V.NONE, V.DEFAULT, V.ALPHA_TEXTURE, V.ALPHA_PROCEDURAL, V.COUNT,
                  V.COUNT_ALPHA_TEXTURE):
            h, which, c = run(V, g, rays.data, q, k)
            ok = okind(V, o, k)
            hit = h["prim"] != MISS
            glob = h.copy()
            glob["prim"] = np.where(hit, offs[np.minimum(which, parts - 1)] + h["prim"], MISS)
            ref, nt = o.trace(cat, rays.data, oq, ok, ties=True)
            compare(o, cat, rays.data, oq, ok, glob, ref, nt)
            wh, ww, wc = o.walk_list(bs, rays.data, oq, ok)
            assert h.tobytes() == wh.tobytes() and np.array_equal(which, ww)
            if c is not None:
                for f in ("boxes", "tris", "alpha"):
                    assert np.array_equal(c[f], wc[f])
    g.close()


def test_group_of_forest_quadrants_matches_single_bvh(V):
    """The C2 forest split into 4 BVHs gives the same closest hits as one BVH
    (up to exact ties) — the list query is the paper's multi-root hierarchy."""
    sc, rays = W.config("C2")
    one = V.Scene.from_workload(sc).build()
    subs = W.split_scene(sc, 4)
    g = V.Group([V.Scene.from_workload(s).build() for s in subs])
    _, offs = W.concat_scenes(subs)
    r = torch.from_numpy(rays.data).cuda()
    ha, _ = one.trace(r, V.CLOSEST, V.ALPHA_TEXTURE)
    hb, wb, _ = g.trace(r, V.CLOSEST, V.ALPHA_TEXTURE)
    torch.cuda.synchronize()
    a, b = V.hits_to_numpy(ha), V.hits_to_numpy(hb)
    assert np.array_equal(a["t"], b["t"])
    hit = b["prim"] != MISS
    assert np.array_equal(a["prim"] != MISS, hit)
    # map (part, local prim) back to the original triangle index
    orig = np.full(len(b), MISS, np.uint64)
    for j, s in enumerate(subs):
        m = hit & (wb.cpu().numpy() == j)
        orig[m] = s.source_index[b["prim"][m]]
    same = orig[hit] == a["prim"][hit]
    assert same.mean() > 0.999   # the rest are exact ties (shared quad diagonals)
    g.close()


def test_group_errors(V):
    sc = W.quad_pair_scene()
    s = V.Scene.from_workload(sc)
    with pytest.raises(V.VsrError) as e:
        V.Group([s])          # not built
    assert e.value.status == V.ERR_NOT_BUILT
    s.build()
    g = V.Group([s, s])
    r = torch.zeros((4, 8), device="cuda")
    with pytest.raises(V.VsrError) as e:
        g.trace(r, V.CLOSEST, V.RUNTIME_SWITCH_DEFAULT)
    assert e.value.status == V.ERR_UNSUPPORTED


@pytest.mark.parametrize("k", [1, 4, 16])
def test_group_multi_vs_walker(V, oracle_lib, k):
    """vsr_trace_group_multi: hits, kept counts, per-hit list index and counts bit-exact vs
    walker C's multi-hit over the list."""
    o = oracle_lib
    sc = W.random_soup(1500, seed=90, size=3.0)
    rays = W.random_rays(3001, seed=91)
    subs = W.split_scene(sc, 4)
    scenes = [V.Scene.from_workload(s).build() for s in subs]
    g = V.Group(scenes)
    bs = [bvh_check.to_oracle(s.export()) for s in scenes]
    r = torch.from_numpy(rays.data).cuda()
    for kind, ok in ((V.ALPHA_TEXTURE, o.ALPHA_TEX), (V.COUNT, o.DEFAULT),
                     (V.ALPHA_PROCEDURAL, o.ALPHA_PROC)):
        h, n, w, c = g.trace_multi(r, k, kind)
        torch.cuda.synchronize()
        wh, wn, ww, wc = o.walk_list_multi(bs, rays.data, k, ok)
        assert np.array_equal(V.hits_to_numpy(h.reshape(-1, 4)).view(np.uint32),
                              wh.reshape(-1).view(np.uint32))
        assert np.array_equal(n.cpu().numpy().astype(np.uint32), wn)
        assert np.array_equal(w.cpu().numpy().astype(np.uint32), ww)
        if c is not None:
            cc = V.counts_to_numpy(c)
            assert np.array_equal(cc["boxes"], wc["boxes"]) and np.array_equal(cc["tris"], wc["tris"])
