"""Pins for the CPU oracle (oracle S, oracle BVH, walker C) — CPU only.

Every check here ties the oracle to something other than itself: the worked
examples of tests/golden/worked_examples.json (each cited), closed forms
computed independently in double precision, invariants of the plain
definition, and hand-built BVHs whose counts are worked
out by hand.  A plausible mistake anywhere in the oracle (a dropped term, a
wrong sign, swapped u/v, a transposed operand, a non-inclusive threshold, a
missing wrap) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
INF = float("inf")


def _ray(lst):
    return np.array([INF if x == "inf" else x for x in lst], dtype=np.float32)


# ----------------------------------------------------------------------------
# Möller–Trumbore
# ----------------------------------------------------------------------------

def test_mt_worked_examples(oracle_lib):
    o = oracle_lib
    tri = GOLD["triangle_cases"]["triangle"]
    for case in GOLD["triangle_cases"]["cases"]:
        hit, t, u, v = o.mt(_ray(case["ray"]), *tri)
        assert hit == case["hit"]
        if hit:
            assert t == case["t"] and u == case["u"] and v == case["v"]


def test_mt_barycentric_convention(oracle_lib):
    """hit point = v0 + u*e1 + v*e2 (reading A10): u belongs to v1, v to v2."""
    v0, v1, v2 = np.array([1.0, 2.0, 3.0]), np.array([4.0, 2.5, 3.0]), np.array([1.5, 6.0, 3.0])
    p = v0 + 0.2 * (v1 - v0) + 0.5 * (v2 - v0)
    ray = np.array([p[0], p[1], 0.0, 1e-4, 0.0, 0.0, 1.0, INF], dtype=np.float32)
    hit, t, u, v = oracle_lib.mt(ray, v0, v1, v2)
    assert hit
    assert abs(u - 0.2) < 1e-6 and abs(v - 0.5) < 1e-6 and abs(t - 3.0) < 1e-6


def test_mt_centroid(oracle_lib):
    v0, v1, v2 = [0, 0, 0], [3, 0, 0], [0, 3, 0]
    ray = np.array([1, 1, -2, 1e-4, 0, 0, 1, INF], dtype=np.float32)
    hit, t, u, v = oracle_lib.mt(ray, v0, v1, v2)
    assert hit and abs(u - 1 / 3) < 1e-6 and abs(v - 1 / 3) < 1e-6 and t == 2.0


def test_mt_interval_inclusive_and_parallel(oracle_lib):
    o = oracle_lib
    tri = ([0, 0, 0], [1, 0, 0], [0, 1, 0])
    # t exactly tmin and exactly tmax are hits ("t in [tmin, tmax]")
    assert o.mt(np.array([.25, .25, -1, 1.0, 0, 0, 1, INF], np.float32), *tri)[0]
    assert o.mt(np.array([.25, .25, -1, 1e-4, 0, 0, 1, 1.0], np.float32), *tri)[0]
    assert not o.mt(np.array([.25, .25, -1, 1e-4, 0, 0, 1, 0.999], np.float32), *tri)[0]
    assert not o.mt(np.array([.25, .25, -1, 1.001, 0, 0, 1, INF], np.float32), *tri)[0]
    # ray parallel to the plane: |det| < 1e-12 -> miss
    assert not o.mt(np.array([.25, .25, 0, 1e-4, 1, 0, 0, INF], np.float32), *tri)[0]
    # behind the origin -> miss
    assert not o.mt(np.array([.25, .25, 1, 1e-4, 0, 0, 1, INF], np.float32), *tri)[0]
    # the barycentric range is closed ("u >= 0, v >= 0, u+v <= 1"): rays exactly
    # on the three edges (values exact in fp32 here) hit
    for x, y in ((0.5, 0.5), (0.0, 0.5), (0.5, 0.0), (0.0, 0.0)):
        hit, t, u, v = o.mt(np.array([x, y, -1, 1e-4, 0, 0, 1, INF], np.float32), *tri)
        assert hit and u == x and v == y, (x, y)
    assert not o.mt(np.array([0.5, 0.5000001, -1, 1e-4, 0, 0, 1, INF], np.float32), *tri)[0]


def _plane_halfplane(ray, vt):
    """Independent double-precision test: plane intersection, then inside test
    with edge half-planes (SPEC S:117 'plane intersection via normal +
    half-plane inside tests').  Returns (hit, t, margin)."""
    o = ray[0:3].astype(np.float64)
    d = ray[4:7].astype(np.float64)
    a, b, c = (vt[0:3].astype(np.float64), vt[3:6].astype(np.float64), vt[6:9].astype(np.float64))
    n = np.cross(b - a, c - a)
    den = n @ d
    if den == 0.0:
        return False, 0.0, 0.0
    t = (n @ (a - o)) / den
    p = o + t * d
    nn = n @ n
    w0 = (np.cross(b - a, p - a) @ n) / nn   # barycentric of c
    w1 = (np.cross(c - b, p - b) @ n) / nn   # barycentric of a
    w2 = (np.cross(a - c, p - c) @ n) / nn   # barycentric of b
    margin = min(w0, w1, w2)
    inside = margin >= 0
    return inside and ray[3] <= t <= ray[7], t, margin


def test_mt_vs_plane_halfplane_10k(oracle_lib):
    rng = np.random.default_rng(1234)
    n = 10000
    agree = 0
    skipped = 0
    for _ in range(n):
        vt = rng.uniform(-2, 2, 9).astype(np.float32)
        o = rng.uniform(-4, 4, 3)
        target = vt[0:3] * 0.4 + vt[3:6] * 0.35 + vt[6:9] * 0.25 + rng.normal(scale=0.8, size=3)
        d = target - o
        ray = np.array([*o, 1e-4, *d, INF], dtype=np.float32)
        hit, t, u, v = oracle_lib.mt(ray, vt[0:3], vt[3:6], vt[6:9])
        rh, rt, margin = _plane_halfplane(ray, vt)
        if abs(margin) < 1e-4 or abs(rt - 1e-4) < 1e-4:
            skipped += 1
            continue
        assert hit == rh
        if hit:
            assert abs(t - rt) <= 1e-5 * abs(rt) + 1e-6
        agree += 1
    assert agree > 9000 and skipped < 1000


def test_mt_translation_invariance(oracle_lib):
    rng = np.random.default_rng(7)
    for _ in range(200):
        vt = rng.uniform(-1, 1, 9)
        o = rng.uniform(-3, 3, 3)
        d = (vt[0:3] + vt[3:6] + vt[6:9]) / 3 - o
        off = rng.uniform(-4, 4, 3)
        r1 = np.array([*o, 1e-4, *d, INF], np.float32)
        r2 = np.array([*(o + off), 1e-4, *d, INF], np.float32)
        vt2 = vt + np.tile(off, 3)
        h1 = oracle_lib.mt(r1, vt[0:3], vt[3:6], vt[6:9])
        h2 = oracle_lib.mt(r2, vt2[0:3], vt2[3:6], vt2[6:9])
        assert h1[0] == h2[0]
        if h1[0]:
            assert abs(h1[1] - h2[1]) <= 1e-4 * abs(h1[1])


# ----------------------------------------------------------------------------
# lerp, tex2D, threshold, procedural
# ----------------------------------------------------------------------------

def test_lerp_worked_examples(oracle_lib):
    g = GOLD["lerp_cases"]
    for u, v, want in g["cases"]:
        got = oracle_lib.lerp2(g["a"], g["b"], g["c"], u, v)
        assert np.allclose(got, want, atol=1e-7)
    # affine identity with a non-trivial triangle: lerp = a + u(b-a) + v(c-a)
    a, b, c = np.array([0.3, -1.0]), np.array([2.0, 0.5]), np.array([-0.7, 4.0])
    got = oracle_lib.lerp2(a, b, c, 0.3, 0.45)
    assert np.allclose(got, a + 0.3 * (b - a) + 0.45 * (c - a), atol=1e-6)


def test_tex2d_worked_examples(oracle_lib):
    g = GOLD["tex2d_cases"]
    rows = np.array(g["texture_2x2_alpha_rows"], dtype=np.uint8)
    tex = np.zeros((2, 2, 4), dtype=np.uint8)
    tex[..., 3] = rows
    for s, t, a8 in g["cases"]:
        assert oracle_lib.tex_alpha(tex, s, t) == np.float32(a8) / np.float32(255.0)


def test_tex2d_1x1_and_wrap(oracle_lib):
    rng = np.random.default_rng(3)
    one = np.array([[[1, 2, 3, 77]]], dtype=np.uint8)
    big = rng.integers(0, 256, (16, 32, 4)).astype(np.uint8)
    for _ in range(500):
        s, t = rng.uniform(-5, 5, 2)
        assert oracle_lib.tex_alpha(one, s, t) == np.float32(77) / np.float32(255)
        k, m = rng.integers(-3, 4, 2)
        # wrap: integer shifts of the coordinate land on the same texel; use
        # coordinates on the dyadic grid so that s+k is exact in fp32
        s2 = np.float32(np.round(s * 64) / 64 + 1 / 128)
        t2 = np.float32(np.round(t * 64) / 64 + 1 / 128)
        assert oracle_lib.tex_alpha(big, s2, t2) == oracle_lib.tex_alpha(big, s2 + k, t2 + m)
        # nearest texel by hand (row j = floor(t*H) mod H, column i = floor(s*W) mod W)
        i = int(math.floor(float(s2) * 32)) % 32
        j = int(math.floor(float(t2) * 16)) % 16
        assert oracle_lib.tex_alpha(big, s2, t2) == np.float32(big[j, i, 3]) / np.float32(255)


def _alpha_scene(a8):
    """One unit quad (2 triangles) at z=1 with a constant-alpha 4x4 texture."""
    sc = W.stacked_quads(1)
    tex = np.full((4, 4, 4), 200, dtype=np.uint8)
    tex[..., 3] = a8
    sc.textures = [tex]
    return sc


def test_alpha_threshold_inclusive(oracle_lib):
    ray = np.array([0.3, 0.6, 0.0, 1e-4, 0, 0, 1, INF], np.float32)
    for a8, keep in GOLD["alpha_a8_decisions"]["cases"]:
        sc = _alpha_scene(a8)
        h = oracle_lib.trace(sc, ray[None], isect=oracle_lib.ALPHA_TEX)
        assert (h["prim"][0] != 0xFFFFFFFF) == keep, a8
        assert (np.float32(a8) / np.float32(255) >= np.float32(GOLD["alpha_threshold"]["value"])) == keep
    # inclusive at equality: threshold exactly a8/255 keeps a8 and rejects a8 - 1
    for a8 in (3, 128, 255):
        thr = float(np.float32(a8) / np.float32(255))
        for val, keep in ((a8, True), (a8 - 1, False)):
            h = oracle_lib.trace(_alpha_scene(val), ray[None], isect=oracle_lib.ALPHA_TEX,
                                 alpha_threshold=thr)
            assert (h["prim"][0] != 0xFFFFFFFF) == keep, (a8, val)


def _hit_at_bary(u, v):
    """Scene + ray hitting the unit right triangle at barycentrics (u, v)."""
    vt = np.array([[0, 0, 1, 1, 0, 1, 0, 1, 1]], dtype=np.float32)
    sc = W.Scene("one", vt, np.zeros(1, np.uint32), np.zeros((1, 6), np.float32),
                 np.zeros(1, np.uint32), [W.gen.white_texture()])
    ray = np.array([u, v, 0.0, 1e-4, 0, 0, 1, INF], np.float32)
    return sc, ray


def test_procedural_worked_examples(oracle_lib):
    for c in GOLD["procedural_cases"]["cases"]:
        sc, ray = _hit_at_bary(c["u"], c["v"])
        acc, t, u, v = oracle_lib.eval_pair(sc, ray, 0, oracle_lib.ALPHA_PROC, checker_freq=c["M"])
        assert acc == c["keep"], c
        assert oracle_lib.eval_pair(sc, ray, 0, oracle_lib.DEFAULT)[0]


# ----------------------------------------------------------------------------
# queries
# ----------------------------------------------------------------------------

def test_stacked_quads_closest(oracle_lib):
    sc = W.stacked_quads(5)
    rays = np.array([[0.3, 0.6, 0, 1e-4, 0, 0, 1, INF], [0.7, 0.2, 0, 1e-4, 0, 0, 1, INF],
                     [0.3, 0.6, 10, 1e-4, 0, 0, -1, INF]], np.float32)
    h = oracle_lib.trace(sc, rays)
    assert h["t"][0] == GOLD["stacked_quads"]["closest_t"] and h["prim"][0] in (0, 1)
    assert h["t"][1] == 1.0 and h["prim"][1] in (0, 1)
    assert h["t"][2] == 5.0 and h["prim"][2] in (8, 9)     # from behind: z=5 first
    # the upper-left point (0.3, 0.6) lies in the second triangle of each quad
    assert h["prim"][0] == 1 and h["prim"][1] == 0


def test_miss_record(oracle_lib):
    sc = W.stacked_quads(2)
    h = oracle_lib.trace(sc, np.array([[5, 5, 0, 1e-4, 0, 0, 1, INF]], np.float32))
    assert h["prim"][0] == 0xFFFFFFFF and h["t"][0] == INF and h["u"][0] == 0 and h["v"][0] == 0


def test_transparent_billboard_passthrough(oracle_lib):
    """A fully transparent quad in front of an opaque one: every interior ray
    returns the back quad (PAPER.md:13-15 'conditionally continue')."""
    sc = W.stacked_quads(2)
    clear = np.zeros((4, 4, 4), np.uint8)
    opaque = np.full((4, 4, 4), 255, np.uint8)
    sc.textures = [clear, opaque]
    sc.geom_texture = np.array([0, 1], np.uint32)
    rng = np.random.default_rng(5)
    xy = rng.uniform(0.01, 0.99, (300, 2))
    rays = np.zeros((300, 8), np.float32)
    rays[:, 0:2] = xy
    rays[:, 3] = 1e-4
    rays[:, 6] = 1
    rays[:, 7] = INF
    for q in (oracle_lib.CLOSEST, oracle_lib.ANY):
        h = oracle_lib.trace(sc, rays, query=q, isect=oracle_lib.ALPHA_TEX)
        assert np.all(h["t"] == 2.0) and np.all(np.isin(h["prim"], [2, 3]))
    hd = oracle_lib.trace(sc, rays, isect=oracle_lib.DEFAULT)
    assert np.all(hd["t"] == 1.0)


def test_masking_only_clears_hits(oracle_lib):
    """Masks only turn hits into misses; accepted hits keep t,u,v,ids; opaque
    texture == DEFAULT; transparent texture == all miss; M=1 == DEFAULT."""
    sc = W.random_soup(300, seed=11)
    rays = W.random_rays(2000, seed=12)
    d = oracle_lib.trace(sc, rays, isect=oracle_lib.DEFAULT)
    for isect in (oracle_lib.ALPHA_TEX, oracle_lib.ALPHA_PROC):
        a = oracle_lib.trace(sc, rays, isect=isect)
        ahit = a["prim"] != 0xFFFFFFFF
        dhit = d["prim"] != 0xFFFFFFFF
        assert np.all(dhit[ahit])                    # alpha hit mask ⊆ default hit mask
        assert np.all(a["t"][ahit] >= d["t"][ahit])  # closest accepted cannot be nearer
        same = a["prim"] == d["prim"]
        assert np.all(a["t"][same] == d["t"][same])
    opaque = W.random_soup(300, seed=11)
    opaque.textures = [np.full((8, 8, 4), 255, np.uint8)] * 2
    a = oracle_lib.trace(opaque, rays, isect=oracle_lib.ALPHA_TEX)
    assert np.array_equal(a, d)
    clear = W.random_soup(300, seed=11)
    clear.textures = [np.zeros((8, 8, 4), np.uint8)] * 2
    a = oracle_lib.trace(clear, rays, isect=oracle_lib.ALPHA_TEX)
    assert np.all(a["prim"] == 0xFFFFFFFF)
    p1 = oracle_lib.trace(sc, rays, isect=oracle_lib.ALPHA_PROC, checker_freq=1)
    assert np.array_equal(p1, d)
    none = oracle_lib.trace(sc, rays, isect=oracle_lib.NONE)
    cnt = oracle_lib.trace(sc, rays, isect=oracle_lib.COUNT)
    assert np.array_equal(none, d) and np.array_equal(cnt, d)


def test_two_pass_equivalence(oracle_lib):
    """In-loop filtering == (all geometric hits) then (filter) then (argmin):
    the 'conditional continue' semantics, checked per ray by brute force."""
    sc = W.random_soup(60, seed=21)
    rays = W.random_rays(200, seed=22)
    for isect in (oracle_lib.ALPHA_TEX, oracle_lib.ALPHA_PROC):
        h = oracle_lib.trace(sc, rays, isect=isect)
        for r in range(rays.n):
            best = (INF, 0xFFFFFFFF)
            for i in range(sc.num_tris):
                geo = oracle_lib.eval_pair(sc, rays.data[r], i, oracle_lib.DEFAULT)
                if not geo[0]:
                    continue
                if not oracle_lib.eval_pair(sc, rays.data[r], i, isect)[0]:
                    continue
                if geo[1] < best[0]:
                    best = (geo[1], i)
            assert h["prim"][r] == best[1] and (best[1] == 0xFFFFFFFF or h["t"][r] == best[0])


def test_permutation_invariance(oracle_lib):
    sc = W.random_soup(400, seed=31)
    rays = W.random_rays(3000, seed=32)
    perm = np.random.default_rng(33).permutation(sc.num_tris)
    sp = W.Scene("perm", sc.vertices[perm], sc.geom_ids[perm], sc.texcoords[perm],
                 sc.geom_texture, sc.textures)
    for isect in (oracle_lib.DEFAULT, oracle_lib.ALPHA_TEX, oracle_lib.ALPHA_PROC):
        a, ta = oracle_lib.trace(sc, rays, isect=isect, ties=True)
        b = oracle_lib.trace(sp, rays, isect=isect)
        hit = b["prim"] != 0xFFFFFFFF
        mapped = np.where(hit, perm[np.minimum(b["prim"], sc.num_tris - 1)], 0xFFFFFFFF)
        ok = ta <= 1
        assert np.array_equal(a["t"], b["t"])
        assert np.array_equal(a["prim"][ok], mapped[ok])


def test_any_query_semantics(oracle_lib):
    sc = W.random_soup(300, seed=41)
    rays = W.random_rays(2000, seed=42)
    for isect in (oracle_lib.DEFAULT, oracle_lib.ALPHA_TEX, oracle_lib.ALPHA_PROC):
        c = oracle_lib.trace(sc, rays, query=oracle_lib.CLOSEST, isect=isect)
        a = oracle_lib.trace(sc, rays, query=oracle_lib.ANY, isect=isect)
        assert np.array_equal(c["prim"] != 0xFFFFFFFF, a["prim"] != 0xFFFFFFFF)
        for r in np.nonzero(a["prim"] != 0xFFFFFFFF)[0][:200]:
            acc, t, u, v = oracle_lib.eval_pair(sc, rays.data[r], a["prim"][r], isect)
            assert acc and t == a["t"][r] and u == a["u"][r] and v == a["v"][r]
            assert t >= c["t"][r]


# ----------------------------------------------------------------------------
# C1 closed form, computed in double here
# ----------------------------------------------------------------------------

def _c1_expected(x, y, tex, alpha_on):
    def alpha_ok(s, t):
        i = int(math.floor(s * 16)) % 16
        j = int(math.floor(t * 16)) % 16
        return (not alpha_on) or tex[j, i, 3] >= 3

    # quad A: [0,1]x[0,.75] at z=1, tc (x, y/.75); tri 0 below diagonal y=.75x
    if 0 <= x <= 1 and 0 <= y <= 0.75:
        s, t = x, y / 0.75
        if alpha_ok(s, t):
            if y <= 0.75 * x:       # tri 0 = (p00, p10, p11)
                v = y / 0.75
                return 1.0, 0, x - v, v
            return 1.0, 1, x, (y - 0.75 * x) / 0.75   # tri 1 = (p00, p11, p01)
    # quad B: [-.5,1.5]x[-.5,1.25] at z=2, tc 2*(p - lo)/extent
    xb, yb = x + 0.5, y + 0.5
    if 0 <= xb <= 2 and 0 <= yb <= 1.75:
        s, t = xb, yb / 1.75 * 2
        if alpha_ok(s, t):
            if yb <= 0.875 * xb:
                v = yb / 1.75
                return 2.0, 2, xb / 2 - v, v
            return 2.0, 3, xb / 2, (yb - 0.875 * xb) / 1.75
    return INF, 0xFFFFFFFF, 0.0, 0.0


def test_c1_closed_form(oracle_lib):
    sc = W.quad_pair_scene()
    rays = W.quad_pair_rays()
    tex = sc.textures[0]
    # generator margins (asserted in double): >= 1e-3 texel from texel lines,
    # >= 1e-4 from quad edges and diagonals
    for x, y in rays.data[:, 0:2].astype(np.float64):
        for s, t in ((x, y / 0.75), (x + 0.5, (y + 0.5) / 1.75 * 2)):
            for q in (s * 16, t * 16):
                assert abs(q - round(q)) > 1e-3
        assert abs(y - 0.75 * x) > 1e-4 and abs((y + .5) - 0.875 * (x + .5)) > 1e-4
    for isect, alpha_on in ((oracle_lib.DEFAULT, False), (oracle_lib.ALPHA_TEX, True)):
        h = oracle_lib.trace(sc, rays, isect=isect)
        n_hit = 0
        for r in range(rays.n):
            x, y = float(rays.data[r, 0]), float(rays.data[r, 1])
            t, prim, u, v = _c1_expected(x, y, tex, alpha_on)
            assert h["prim"][r] == prim, (r, x, y)
            if prim != 0xFFFFFFFF:
                n_hit += 1
                assert h["t"][r] == t
                assert abs(h["u"][r] - u) < 1e-6 and abs(h["v"][r] - v) < 1e-6
        assert 0 < n_hit < rays.n


# ----------------------------------------------------------------------------
# walker C (contract traversal) and the oracle BVH
# ----------------------------------------------------------------------------

def test_slab_worked_examples(oracle_lib):
    g = GOLD["slab_cases"]
    lo, hi = g["box"]
    for c in g["cases"]:
        hit, tn, tf = oracle_lib.slab(lo, hi, _ray(c["ray"]))
        assert hit == c["hit"]
        if hit:
            assert tn == c["tnear"]
            assert c["tfar"] <= tf <= c["tfar"] * (1 + 4e-7)
    # origin inside: tnear clipped to tmin, tfar > 0
    hit, tn, tf = oracle_lib.slab(lo, hi, np.array([0, 0, 0, 1e-4, 0.3, -0.2, 1, INF], np.float32))
    assert hit and tn == np.float32(1e-4) and tf > 0
    # zero direction components stay NaN-free (guarded reciprocal, reading A20)
    hit, tn, tf = oracle_lib.slab(lo, hi, np.array([0.5, 0.5, -3, 1e-4, 0, 0, 1, INF], np.float32))
    assert hit and not math.isnan(tn) and not math.isnan(tf)
    # best_t clip: box farther than the current best -> miss
    hit, _, _ = oracle_lib.slab(lo, hi, _ray(g["cases"][0]["ray"]), best_t=0.5)
    assert not hit


@pytest.mark.parametrize("max_leaf", [1, 4, 16])
def test_oracle_bvh_valid(oracle_lib, max_leaf):
    from tests import bvh_check
    sc = W.random_soup(777, seed=51)
    b = oracle_lib.build_bvh(sc, max_leaf)
    bvh_check.validate(b, sc.vertices, max_leaf)
    assert b.tris.shape[0] == 777


def _hand_bvh(z_left=1.0, z_right=3.0, transparent_left=False):
    """Hand-built export arrays: root inner node with two leaves, each leaf one
    unit quad (2 triangles) — left at z_left, right at z_right."""
    f = np.float32
    nodes = np.zeros((1, 16), np.uint32)
    nf = nodes.view(np.float32)
    # per axis k: (lo0.k, lo1.k, hi0.k, hi1.k); child 0 at z_left, child 1 at z_right (flat in z)
    nf[0, 0:4] = [0, 0, 1, 1]
    nf[0, 4:8] = [0, 0, 1, 1]
    nf[0, 8:12] = [z_left, z_right, z_left, z_right]
    LEAF = 0x80000000
    nodes[0, 12] = LEAF | (1 << 26) | 0           # leaf: 2 tris from 0
    nodes[0, 13] = LEAF | (1 << 26) | 2           # leaf: 2 tris from 2
    tris = np.zeros((4, 12), np.uint32)
    tf_ = tris.view(np.float32)
    sides = np.zeros((4, 8), np.uint32)
    sf = sides.view(np.float32)
    for q, z in enumerate((z_left, z_right)):
        for k, (e1, e2) in enumerate((([1, 0, 0], [1, 1, 0]), ([1, 1, 0], [0, 1, 0]))):
            i = 2 * q + k
            tf_[i, 0:3] = [0, 0, z]
            tris[i, 3] = i
            tf_[i, 4:7] = e1
            tf_[i, 8:11] = e2
            sf[i, 0:6] = [0, 0, 1, 0, 1, 1] if k == 0 else [0, 0, 1, 1, 0, 1]
            # sidecar word 6 = first texel of the texture, word 7 = (W-1)|(H-1)<<16 (1x1)
            sides[i, 6] = 0 if (q == 0 and transparent_left) else 1
            sides[i, 7] = 0
    texdescs = np.array([[0, 0, 1, 1], [1, 0, 1, 1]], np.uint32)
    texels = np.array([0, 255], np.uint8)          # A8 plane: transparent, opaque
    return oracle_lib_bvh(0, np.array([0, 0, min(z_left, z_right)], f),
                          np.array([1, 1, max(z_left, z_right)], f), nodes, tris, sides, texdescs,
                          texels)


def oracle_lib_bvh(*a):
    import oracle
    return oracle.BvhArrays(*a)


def test_walker_hand_counts(oracle_lib):
    o = oracle_lib
    b = _hand_bvh()
    R = lambda *r: np.array([r], np.float32)  # noqa: E731
    # +z through both quads: root(1) + node(2); near leaf (2 tris); far entry
    # popped with tnear 3 > best_t 1 -> skipped without a hook call.
    h, c = o.walk(b, R(.25, .75, 0, 1e-4, 0, 0, 1, INF), isect=o.COUNT)
    assert (c["boxes"][0], c["tris"][0]) == (3, 2) and h["t"][0] == 1.0 and h["prim"][0] == 1
    # -z from behind: the right child is nearer and is visited first
    h, c = o.walk(b, R(.25, .75, 5, 1e-4, 0, 0, -1, INF), isect=o.COUNT)
    assert (c["boxes"][0], c["tris"][0]) == (3, 2) and h["t"][0] == 2.0 and h["prim"][0] == 3
    # root miss -> (1, 0)
    h, c = o.walk(b, R(5, 5, 0, 1e-4, 0, 0, 1, INF), isect=o.COUNT)
    assert (c["boxes"][0], c["tris"][0]) == (1, 0) and h["prim"][0] == 0xFFFFFFFF
    # transparent near quad: traversal continues into the far leaf (4 tests)
    bt = _hand_bvh(transparent_left=True)
    h, c = o.walk(bt, R(.25, .75, 0, 1e-4, 0, 0, 1, INF), isect=o.ALPHA_TEX)
    assert (c["boxes"][0], c["tris"][0], c["alpha"][0]) == (3, 4, 2)
    assert h["t"][0] == 3.0 and h["prim"][0] == 3
    # ANY stops at the first accepted hit: near leaf, first triangle that hits
    h, c = o.walk(b, R(.75, .25, 0, 1e-4, 0, 0, 1, INF), query=o.ANY, isect=o.COUNT)
    assert (c["boxes"][0], c["tris"][0]) == (3, 1) and h["prim"][0] == 0


def test_walker_single_leaf_counts(oracle_lib):
    for k in (1, 3, 4):
        sc = W.stacked_quads(4)
        sc = W.Scene("k", sc.vertices[:k], sc.geom_ids[:k], sc.texcoords[:k], sc.geom_texture,
                     sc.textures)
        b = oracle_lib.build_bvh(sc, max_leaf=4)
        assert b.nodes.shape[0] == 0 and b.root_ref & 0x80000000
        rays = np.array([[0.5, 0.5, -1, 1e-4, 0, 0, 1, INF]], np.float32)
        _, c = oracle_lib.walk(b, rays, isect=oracle_lib.COUNT)
        assert (c["boxes"][0], c["tris"][0]) == (1, k)


@pytest.mark.parametrize("max_leaf", [1, 4, 16])
def test_walker_equals_bruteforce(oracle_lib, max_leaf):
    o = oracle_lib
    sc = W.random_soup(500, seed=61 + max_leaf)
    rays = W.random_rays(3000, seed=62)
    b = o.build_bvh(sc, max_leaf)
    for isect in (o.DEFAULT, o.ALPHA_TEX, o.ALPHA_PROC):
        s, nt = o.trace(sc, rays, isect=isect, ties=True)
        w, c = o.walk(b, rays, isect=isect)
        assert np.array_equal(s["t"], w["t"])
        ok = nt <= 1
        assert np.array_equal(s["prim"][ok], w["prim"][ok])
        assert np.array_equal(s["u"][ok], w["u"][ok]) and np.array_equal(s["v"][ok], w["v"][ok])
        # counting invariants: boxes = 1 + 2*inner visited (odd),
        # boxes <= 2*nodes + 1, tris <= N
        assert np.all(c["boxes"] % 2 == 1)
        assert np.all(c["boxes"] <= 2 * b.nodes.shape[0] + 1)
        assert np.all(c["tris"] <= sc.num_tris)
        assert np.all(c["tris"][w["prim"] != 0xFFFFFFFF] >= 1)
        wa, ca = o.walk(b, rays, query=o.ANY, isect=isect)
        assert np.array_equal(wa["prim"] != 0xFFFFFFFF, s["prim"] != 0xFFFFFFFF)
        assert np.all(ca["tris"] <= c["tris"])


def test_walker_c1(oracle_lib):
    o = oracle_lib
    sc = W.quad_pair_scene()
    rays = W.quad_pair_rays()
    b = o.build_bvh(sc, 1)
    for isect in (o.DEFAULT, o.ALPHA_TEX, o.ALPHA_PROC):
        s = o.trace(sc, rays, isect=isect)
        w, _ = o.walk(b, rays, isect=isect)
        assert np.array_equal(s, w)


def test_flags_near_tie(oracle_lib):
    """Two coincident quads -> every interior hit is an exact tie (X1)."""
    sc = W.stacked_quads(2, z0=1.0, dz=0.0)
    rays = np.array([[0.3, 0.4, 0, 1e-4, 0, 0, 1, INF], [0.9, 0.05, 0, 1e-4, 0, 0, 1, INF]],
                    np.float32)
    h, fl, nt = oracle_lib.trace(sc, rays, flags=True, ties=True)
    assert np.all(fl & oracle_lib.X1) and np.all(nt == 2)
    assert np.all(h["prim"] == np.array([1, 0]))  # lowest index wins exact ties
