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


# ---- conservativeness against exact rational arithmetic (the definition of a hit) ----------
from fractions import Fraction as Fr  # noqa: E402


def _exact_entry(lo, hi, o, d, tmin, tmax):
    """Exact (rational) intersection of the segment o + t d, t in [tmin, tmax], with the
    closed box [lo, hi]: the entry t, or None if they do not meet."""
    a, b = Fr(float(tmin)), (Fr(float(tmax)) if np.isfinite(tmax) else None)
    for k in range(3):
        ok, dk = Fr(float(o[k])), Fr(float(d[k]))
        lk, hk = Fr(float(lo[k])), Fr(float(hi[k]))
        if dk == 0:
            if not (lk <= ok <= hk):
                return None
            continue
        t0, t1 = (lk - ok) / dk, (hk - ok) / dk
        if t0 > t1:
            t0, t1 = t1, t0
        a = max(a, t0)
        b = t1 if b is None else min(b, t1)
    return a if (b is None or a <= b) else None


def _grazing_cases(n, seed, far):
    """Boxes near the coordinate origin, ray origins `far` away along random directions,
    aimed at points ON the box boundary (edges and corners): the exact segment touches the
    box, so the inclusive test must report a hit.  Non-dyadic directions make inv and
    o * inv inexact."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        c = rng.uniform(-2, 2, 3)
        h = rng.uniform(1e-3, 1.0, 3)
        lo, hi = (c - h).astype(np.float32), (c + h).astype(np.float32)
        p = rng.uniform(lo, hi)
        snap = rng.integers(1, 4)   # snap 1..3 coordinates to the boundary: faces, edges, corners
        for k in rng.choice(3, snap, replace=False):
            p[k] = lo[k] if rng.random() < 0.5 else hi[k]
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        o = (p + far * u).astype(np.float32)
        d = ((p - o) * rng.uniform(0.3, 3.0)).astype(np.float32)
        out.append((lo, hi, o, d))
    return out


@pytest.mark.parametrize("far", [3.0, 1e3, 1e6])
def test_slab_conservative_vs_exact(far):
    """Every box the exact segment meets is reported hit by the fp32 test (tmax = +inf)."""
    met = 0
    for lo, hi, o, d in _grazing_cases(600, int(far) + 3, far):
        if _exact_entry(lo, hi, o, d, np.float32(1e-4), np.inf) is None:
            continue
        met += 1
        hit, _, _ = oracle.slab(lo, hi, np.array([*o, 1e-4, *d, np.inf], np.float32))
        assert hit, (lo, hi, o, d)
    assert met > 100


@pytest.mark.parametrize("far", [1e3, 1e6])
def test_slab_best_t_bound_conservative(far):
    """A box whose exact entry t* is <= best_t must not be culled: best_t = the float just
    at or above t* (the tightest admissible bound), rays whose origin term o*inv is large
    against t* (the fma form's absolute error e is then far above u t*)."""
    met = 0
    for lo, hi, o, d in _grazing_cases(600, int(far) + 7, far):
        t_star = _exact_entry(lo, hi, o, d, np.float32(1e-4), np.inf)
        if t_star is None or t_star <= 0:
            continue
        bt = np.float32(float(t_star))
        if Fr(float(bt)) < t_star:
            bt = np.nextafter(bt, np.float32(np.inf))
        met += 1
        hit, _, _ = oracle.slab(lo, hi, np.array([*o, 1e-4, *d, np.inf], np.float32), best_t=float(bt))
        assert hit, (lo, hi, o, d, float(bt))
    assert met > 100


def _rn32(x):
    """Round a rational to the nearest float32 (ties to even), exactly — no double rounding."""
    if x == 0:
        return np.float32(0.0)
    s = -1 if x < 0 else 1
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fr(2) ** e > a:
        e -= 1
    e = max(e, -126)                       # subnormals share the minimum exponent
    scaled = a / Fr(2) ** (e - 23)         # 24-bit mantissa scale
    q, r = divmod(scaled.numerator, scaled.denominator)
    if 2 * r > scaled.denominator or (2 * r == scaled.denominator and q % 2 == 1):
        q += 1
    return np.float32(s * float(Fr(q) * Fr(2) ** (e - 23)))


def test_plane_crossing_is_one_rounding():
    """Contract r02's plane crossing is t = RN(plane * inv + noi) — ONE rounding of the
    exact value (an fma), with noi = RN(-(o * inv)).  Checked on the walker's entry value
    against exact rational arithmetic: tn = max(min over each axis's two planes, tmin)."""
    rng = np.random.default_rng(99)
    checked = 0
    for lo, hi, o, d in _grazing_cases(300, 99, 1e3):
        ray = np.array([*o, 1e-4, *d, np.inf], np.float32)
        inv = [np.float32(1.0) / (d[k] if abs(d[k]) > 2.0 ** -80 else np.copysign(np.float32(2.0 ** -80), d[k]))
               for k in range(3)]
        ts = []
        for k in range(3):
            noi = _rn32(-(Fr(float(o[k])) * Fr(float(inv[k]))))
            a = _rn32(Fr(float(lo[k])) * Fr(float(inv[k])) + Fr(float(noi)))
            b = _rn32(Fr(float(hi[k])) * Fr(float(inv[k])) + Fr(float(noi)))
            ts.append(min(a, b))
        tn_expect = max(max(ts), np.float32(1e-4))
        _, tn, _ = oracle.slab(lo, hi, ray)
        assert np.float32(tn) == tn_expect, (tn, tn_expect)
        checked += 1
    assert checked == 300 and rng is not None
