"""Pins for the list-of-BVHs walker (BVHs as compound
primitives, more than one root) — CPU only."""
import numpy as np
import pytest

import workloads as W

INF = float("inf")
MISS = 0xFFFFFFFF


@pytest.mark.parametrize("parts", [1, 2, 5])
def test_list_walker_equals_bruteforce(oracle_lib, parts):
    o = oracle_lib
    sc = W.random_soup(700, seed=11 + parts)
    rays = W.random_rays(3000, seed=12)
    subs = W.split_scene(sc, parts)
    cat, offs = W.concat_scenes(subs)
    bs = [o.build_bvh(s, 2) for s in subs]
    for isect in (o.DEFAULT, o.ALPHA_TEX, o.ALPHA_PROC):
        ref, nt = o.trace(cat, rays, o.CLOSEST, isect, ties=True)
        h, which, c = o.walk_list(bs, rays, o.CLOSEST, isect)
        hit = h["prim"] != MISS
        assert np.array_equal(hit, ref["prim"] != MISS)
        assert np.array_equal(h["t"], ref["t"])
        glob = np.where(hit, offs[np.minimum(which, parts - 1)] + h["prim"], MISS)
        ok = nt <= 1
        assert np.array_equal(glob[ok], ref["prim"][ok])
        assert np.all(which[~hit] == MISS)
        a, aw, ac = o.walk_list(bs, rays, o.ANY, isect)
        assert np.array_equal(a["prim"] != MISS, hit)
        assert np.all(ac["boxes"] >= parts)          # every root tested once
        assert np.all(ac["tris"] <= c["tris"] + 0)   # any-hit never does more leaf work


def test_single_element_list_is_the_plain_walk(oracle_lib):
    o = oracle_lib
    sc = W.random_soup(500, seed=3)
    rays = W.random_rays(2000, seed=4)
    b = o.build_bvh(sc, 2)
    for q in (o.CLOSEST, o.ANY):
        h1, c1 = o.walk(b, rays, q, o.ALPHA_TEX)
        h2, w2, c2 = o.walk_list([b], rays, q, o.ALPHA_TEX)
        assert np.array_equal(h1, h2) and np.array_equal(c1, c2)
        assert np.all(w2[h2["prim"] != MISS] == 0)


def test_counts_add_over_the_list_and_which(oracle_lib):
    """Two quads in separate single-leaf BVHs (z=1 in element 1, z=2 in element 0)."""
    o = oracle_lib
    near = W.stacked_quads(1, z0=1.0)
    far = W.stacked_quads(1, z0=2.0)
    bs = [o.build_bvh(far, 2), o.build_bvh(near, 2)]
    rays = np.array([[0.3, 0.6, 0, 1e-4, 0, 0, 1, INF],     # through both
                     [5, 5, 0, 1e-4, 0, 0, 1, INF]], np.float32)  # misses both roots
    h, which, c = o.walk_list(bs, rays, o.CLOSEST, o.COUNT)
    assert h["t"][0] == 1.0 and which[0] == 1 and h["prim"][0] == 1
    assert (c["boxes"][0], c["tris"][0]) == (2, 4)    # 2 roots + 2 single-leaf BVHs of 2 tris
    assert (c["boxes"][1], c["tris"][1]) == (2, 0) and which[1] == MISS
    # reversed list: the near quad first prunes the far BVH's root (tn 2 > best_t 1)
    h, which, c = o.walk_list(bs[::-1], rays, o.CLOSEST, o.COUNT)
    assert which[0] == 0 and (c["boxes"][0], c["tris"][0]) == (2, 2)


@pytest.mark.parametrize("parts,k", [(1, 4), (3, 4), (5, 16)])
def test_list_multi_walker_equals_bruteforce(oracle_lib, parts, k):
    """Multi-hit over a list: the walker's k smallest-t accepted hits across
    all elements equal the brute force's on the concatenated triangles (t lists exact, prims up
    to exact ties), and each kept hit's list index maps it back to its element."""
    o = oracle_lib
    sc = W.random_soup(600, seed=30 + parts, size=3.0)
    rays = W.random_rays(2000, seed=31)
    subs = W.split_scene(sc, parts)
    cat, offs = W.concat_scenes(subs)
    bs = [o.build_bvh(s, 2) for s in subs]
    for isect in (o.DEFAULT, o.ALPHA_TEX):
        ref, rn, rc = o.trace_multi(cat, rays, k, isect)
        h, nh, which, c = o.walk_list_multi(bs, rays, k, isect)
        assert np.array_equal(nh, rn)
        assert np.array_equal(h["t"], ref["t"])
        kept = h["prim"] != MISS
        glob = np.where(kept, offs[np.minimum(which, parts - 1)] + h["prim"], MISS)
        # equal t may come in another order: compare per-ray sets of (t, prim)
        for i in np.nonzero((glob != ref["prim"]).any(axis=1))[0]:
            assert sorted(zip(h["t"][i][kept[i]], glob[i][kept[i]])) == \
                sorted(zip(ref["t"][i][kept[i]], ref["prim"][i][kept[i]])) or rc[i] > 0, i
        assert np.all(which[~kept] == MISS)


def test_single_element_list_multi_is_walk_multi(oracle_lib):
    o = oracle_lib
    sc = W.random_soup(500, seed=33)
    rays = W.random_rays(1500, seed=34)
    b = o.build_bvh(sc, 2)
    h1, n1, c1 = o.walk_multi(b, rays, 4, o.ALPHA_TEX)
    h2, n2, w2, c2 = o.walk_list_multi([b], rays, 4, o.ALPHA_TEX)
    assert np.array_equal(h1, h2) and np.array_equal(n1, n2) and np.array_equal(c1, c2)
    assert np.all(w2[h2["prim"] != MISS] == 0)
