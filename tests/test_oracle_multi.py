"""Pins for the multi-hit oracle ("the first N hit points";
SPEC S:285-293) and the multi-hit contract walker — CPU only."""
import json
import os

import numpy as np
import pytest

import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
INF = float("inf")
MISS = 0xFFFFFFFF


def test_stacked_quads_worked_example(oracle_lib):
    g = GOLD["multi_hit_stacked"]
    sc = W.stacked_quads(5)
    rays = np.array([[0.3, 0.6, 0, 1e-4, 0, 0, 1, INF]], np.float32)
    h, nh, _ = oracle_lib.trace_multi(sc, rays, g["k"])
    assert list(h["t"][0]) == g["t"] and nh[0] == g["k"]
    assert list(h["prim"][0]) == [1, 3, 5]          # the upper-left triangle of each quad
    h, nh, _ = oracle_lib.trace_multi(sc, rays, 16)  # more slots than hits
    assert nh[0] == 5 and list(h["t"][0][:5]) == [1, 2, 3, 4, 5]
    assert np.all(h["prim"][0][5:] == MISS) and np.all(h["t"][0][5:] == INF)


def test_all_hits_equal_pairwise_brute_force(oracle_lib):
    """k >= #accepted: the multi list is every accepted candidate, ascending t,
    built here independently from per-pair evaluations."""
    o = oracle_lib
    sc = W.random_soup(120, seed=3, size=4.0)
    rays = W.random_rays(150, seed=4)
    for isect in (o.DEFAULT, o.ALPHA_TEX, o.ALPHA_PROC):
        h, nh, _ = o.trace_multi(sc, rays, 32, isect=isect)
        for r in range(rays.n):
            acc = []
            for i in range(sc.num_tris):
                ok, t, u, v = o.eval_pair(sc, rays.data[r], i, isect)
                if ok:
                    acc.append((t, i))
            acc.sort()
            assert nh[r] == min(len(acc), 32)
            assert [x[0] for x in acc[:32]] == list(h["t"][r][:nh[r]])
            assert [x[1] for x in acc[:32]] == list(h["prim"][r][:nh[r]])


def test_k1_equals_closest(oracle_lib):
    o = oracle_lib
    sc = W.random_soup(400, seed=9)
    rays = W.random_rays(2000, seed=10)
    for isect in (o.DEFAULT, o.ALPHA_TEX):
        c = o.trace(sc, rays, isect=isect)
        m, nh, _ = o.trace_multi(sc, rays, 1, isect=isect)
        assert np.array_equal(m[:, 0], c)
        assert np.array_equal(nh == 1, c["prim"] != MISS)


def test_transparent_front_quad_is_skipped(oracle_lib):
    sc = W.stacked_quads(3)
    sc.textures = [np.zeros((2, 2, 4), np.uint8), np.full((2, 2, 4), 255, np.uint8)]
    sc.geom_texture = np.array([0, 1, 1], np.uint32)
    rays = np.array([[0.7, 0.2, 0, 1e-4, 0, 0, 1, INF]], np.float32)
    h, nh, _ = oracle_lib.trace_multi(sc, rays, 4, isect=oracle_lib.ALPHA_TEX)
    assert nh[0] == 2 and list(h["t"][0][:2]) == [2.0, 3.0]


def _same_up_to_ties(a, na, b, nb):
    """Equal t lists; within each group of equal t the prims may differ only
    where the group is cut by k (checked by the caller via ncut)."""
    assert np.array_equal(na, nb)
    assert np.array_equal(a["t"], b["t"])


@pytest.mark.parametrize("k", [1, 2, 5, 16])
def test_walker_multi_equals_bruteforce(oracle_lib, k):
    o = oracle_lib
    sc = W.random_soup(600, seed=20 + k, size=3.0)
    rays = W.random_rays(2500, seed=30)
    b = o.build_bvh(sc, 2)
    for isect in (o.DEFAULT, o.ALPHA_TEX, o.ALPHA_PROC):
        h, nh, nc = o.trace_multi(sc, rays, k, isect=isect)
        w, wn, wc = o.walk_multi(b, rays, k, isect=isect)
        _same_up_to_ties(h, nh, w, wn)
        # prims agree except inside a tie group cut at the k-th entry
        for r in np.nonzero(np.any(h["prim"] != w["prim"], axis=1))[0]:
            assert nc[r] > 1 or len(set(h["t"][r])) < k
        # counting invariants; k = 1 walks exactly like the closest-hit walker
        assert np.all(wc["boxes"] % 2 == 1)
        if k == 1:
            cw, cc = o.walk(b, rays, isect=isect)
            assert np.array_equal(w[:, 0], cw) and np.array_equal(wc, cc)
