"""Pins for the slab contract r02 (DESIGN.md §3 A.2), CPU only: the box test computes
each plane crossing as ONE fma, t = fma(plane, inv, noi) with noi = -(o*inv), widens
tf by (1 + 2 gamma_3) and by pad = 4 max_k |e_k| (e_k = noi_k's exact rounding error),
and compares tn with best_t + pad.  The fma form's error is ABSOLUTE in |o*inv|, so
rays whose origin is far from the coordinate origin relative to the boxes they test
are where a missing allowance would cull true hits.  Pinned against the plain
definition (oracle S brute force): the BVH only prunes, so walker C's hit/miss must
equal brute force's on every such ray."""
import numpy as np
import pytest

import oracle
import workloads as W


@pytest.fixture(scope="module", autouse=True)
def _lib(oracle_lib):
    return oracle_lib


def _far_rays(tris, n, dist, rng):
    """Rays from origins `dist` away (random directions, non-dyadic) aimed at points
    inside random triangles near their edges/corners, where the boxes are tight."""
    k = rng.integers(0, tris.shape[0], n)
    v = tris[k].reshape(n, 3, 3).astype(np.float64)
    b = rng.dirichlet([0.3, 0.3, 0.3], n)                 # near edges / corners
    p = (b[:, :, None] * v).sum(axis=1)
    u = rng.normal(size=(n, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    o = p + dist * u
    d = (p - o) * rng.uniform(0.3, 3.0, (n, 1))           # unnormalised, inexact inverses
    r = np.zeros((n, 8), np.float32)
    r[:, 0:3] = o
    r[:, 3] = 1e-4
    r[:, 4:7] = d
    r[:, 7] = np.inf
    return r


@pytest.mark.parametrize("dist", [1e2, 1e3, 1e4, 1e5])
@pytest.mark.parametrize("max_leaf", [1, 4])
def test_far_origins_never_culled(dist, max_leaf):
    sc = W.random_soup(200, seed=21, extent=3.0, size=0.8)
    rng = np.random.default_rng(int(dist) + max_leaf)
    rays = _far_rays(sc.vertices, 4000, dist, rng)
    b = oracle.build_bvh(sc, max_leaf)
    wh, _ = oracle.walk(b, rays, oracle.CLOSEST, oracle.DEFAULT)
    ref = oracle.trace(sc, rays, oracle.CLOSEST, oracle.DEFAULT)
    hit_w, hit_r = wh["prim"] != 0xFFFFFFFF, ref["prim"] != 0xFFFFFFFF
    assert hit_r.mean() > 0.5
    assert np.array_equal(hit_w, hit_r), np.nonzero(hit_w != hit_r)[0][:5]
    same = wh["prim"] == ref["prim"]
    assert np.array_equal(wh["t"][same], ref["t"][same])


def test_thin_box_far_origin():
    """A flat triangle (box thickness = the 2^-20 padding only) seen from 1e5 away along
    inexact directions: the z-slab's shift e is far larger than the slab, yet every hit
    must survive the root test and the walk."""
    tri = np.array([[0.1, 0.2, 0.0, 0.9, 0.3, 0.0, 0.2, 0.8, 0.0]], np.float32)
    sc = W.Scene("thin", tri, np.zeros(1, np.uint32), np.zeros((1, 6), np.float32),
                 np.zeros(1, np.uint32), [np.full((1, 1, 4), 255, np.uint8)])
    rng = np.random.default_rng(5)
    rays = _far_rays(tri, 2000, 1e5, rng)
    b = oracle.build_bvh(sc, 1)
    wh, wc = oracle.walk(b, rays, oracle.ANY, oracle.DEFAULT)
    ref = oracle.trace(sc, rays, oracle.ANY, oracle.DEFAULT)
    assert np.array_equal(wh["prim"] != 0xFFFFFFFF, ref["prim"] != 0xFFFFFFFF)
    assert (ref["prim"] != 0xFFFFFFFF).mean() > 0.5


def test_pad_is_zero_for_exact_origin_terms():
    """Axis-parallel and power-of-two directions make noi exact (e = 0): the allowance is
    zero and the test is the old one (S:125-127 worked example: tnear 1, tfar 3 x 1.0000003576)."""
    hit, tn, tf = oracle.slab([-1, -1, -1], [1, 1, 1],
                              np.array([0, 0, -2, 1e-4, 0, 0, 1, np.inf], np.float32))
    assert hit and tn == 1.0 and tf == np.float32(3.0) * np.float32(1.0000003576)


def test_overflowing_origin_term_never_culls():
    """|o * inv| beyond FLT_MAX (origin 1e30 on an axis-parallel component, inv = 2^80):
    noi is clamped, e (hence pad) becomes infinite, the test widens to 'hit' — no NaN."""
    hit, tn, tf = oracle.slab([-1, -1, -1], [1, 1, 1],
                              np.array([1e30, 0, -2, 1e-4, 0, 0, 1, np.inf], np.float32))
    assert hit and not np.isnan(tn) and tf == np.inf
