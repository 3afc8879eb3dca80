"""Pins for oracle S's ambiguity flags X1-X5 (SURVEY.md §8(c) "Ambiguity exclusion
classes"; DESIGN.md §5 and reading A28).  CPU only.

The flags decide which rays the GPU parity tests may exclude, so each class is
pinned here by a closed-form case where the flag MUST fire and a neighbour where
it must NOT (a flag that fires everywhere would hide real mismatches):

* X1 near tie  — two accepted t within 1e-5 relative (north_star);
* X2 edge graze — the double-precision barycentric margin min(u, v, 1-u-v) < 1e-6;
* X3 texel edge — s*W (or t*H) within 1e-5 of an integer AND the texels on either
  side decide differently (an opaque/transparent column pair vs a uniform one);
* X4 checker edge — u*M (or v*M) an integer (ALPHA_PROCEDURAL, M = 8);
* X5 alpha near threshold — the bilinear alpha within the derived band of the
  threshold: north_star's 1e-6 floor (texcoords exact here, so the propagated
  term is 0), exercised at alpha = thr, thr + 4.8e-7 (inside) and thr + 7.6e-6
  (outside).

Geometry: the unit triangle v0 = (0,0,0), v1 = (1,0,0), v2 = (0,1,0) hit by
o = (x, y, -1), d = (0, 0, 1) gives, exactly in fp32 and in double, t = 1,
u = x, v = y (worked by hand: e1 = (1,0,0), e2 = (0,1,0), p = d x e2 = (-1,0,0),
det = -1, u = (s.p)/det = x, q = s x e1 = (0,-1,-y), v = (d.q)/det = y,
t = (e2.q)/det = 1).  Texcoords (0,0), (1,0), (0,1) make (s, t) = (u, v).
"""
import numpy as np
import pytest

import oracle
import workloads as W


def _scene(tris, texture=None):
    tris = np.asarray(tris, dtype=np.float32).reshape(-1, 9)
    n = tris.shape[0]
    tc = np.tile(np.array([0, 0, 1, 0, 0, 1], np.float32), (n, 1))
    tex = texture if texture is not None else np.full((1, 1, 4), 255, np.uint8)
    return W.Scene("flags", tris, np.zeros(n, np.uint32), tc, np.zeros(1, np.uint32), [tex])


UNIT = [0, 0, 0, 1, 0, 0, 0, 1, 0]


def _ray(x, y, z0=-1.0):
    return np.array([[x, y, z0, 1e-4, 0, 0, 1, np.inf]], np.float32)


def _flags(sc, ray, query=oracle.CLOSEST, isect=oracle.DEFAULT, thr=0.01, M=8):
    _, fl = oracle.trace(sc, ray, query, isect, alpha_threshold=thr, checker_freq=M, flags=True,
                         nthreads=1)
    return int(fl[0])


@pytest.fixture(scope="module", autouse=True)
def _lib(oracle_lib):
    return oracle_lib


def test_worked_geometry_is_exact():
    h = oracle.trace(_scene(UNIT), _ray(0.375, 0.25), oracle.CLOSEST, oracle.DEFAULT, nthreads=1)
    assert (h["t"][0], h["u"][0], h["v"][0], h["prim"][0]) == (1.0, 0.375, 0.25, 0)


# ---- X1 near tie (north_star: 1e-5 relative) -------------------------------------
@pytest.mark.parametrize("order", ["near_first", "far_first"])
def test_x1_fires_within_1e_5_relative(order):
    far = [0, 0, 5e-6, 1, 0, 5e-6, 0, 1, 5e-6]    # t = 1 + 5e-6
    tris = UNIT + far if order == "near_first" else far + UNIT
    assert _flags(_scene(tris), _ray(0.3, 0.3)) & oracle.X1


def test_x1_fires_on_exact_tie():
    assert _flags(_scene(UNIT + UNIT), _ray(0.3, 0.3)) & oracle.X1


@pytest.mark.parametrize("order", ["near_first", "far_first"])
def test_x1_silent_when_separated(order):
    far = [0, 0, 1e-3, 1, 0, 1e-3, 0, 1, 1e-3]    # t = 1.001: 1e-3 relative
    tris = UNIT + far if order == "near_first" else far + UNIT
    assert not _flags(_scene(tris), _ray(0.3, 0.3)) & oracle.X1


def test_x1_ignores_vetoed_candidates():
    """A candidate the filter rejects is not in A, so it cannot make a tie: the near
    triangle is transparent under ALPHA_TEX (alpha 0 everywhere on a 1x1 texture)."""
    clear = np.zeros((1, 1, 4), np.uint8)
    tris = UNIT + [0, 0, 5e-6, 1, 0, 5e-6, 0, 1, 5e-6]
    sc = _scene(tris, clear)
    assert not _flags(sc, _ray(0.3, 0.3), isect=oracle.ALPHA_TEX) & oracle.X1


# ---- X2 edge graze (double margin < 1e-6) -------------------------------------------
@pytest.mark.parametrize("x,y", [(0.5, 0.0), (0.0, 0.5), (0.5, 0.5), (0.5, 1e-7),
                                 (0.5, -1e-7), (0.25, 0.75 - 2**-24)])
def test_x2_fires_on_edges(x, y):
    assert _flags(_scene(UNIT), _ray(x, y)) & oracle.X2


@pytest.mark.parametrize("x,y", [(0.25, 0.25), (0.5, 1e-5), (0.5, -1e-5), (0.3, 0.6)])
def test_x2_silent_inside_and_outside(x, y):
    assert not _flags(_scene(UNIT), _ray(x, y)) & oracle.X2


# ---- X3 texel edge with straddling texels ------------------------------------------
def _columns(a_left, a_right):
    """2x2 RGBA8: column 0 alpha a_left, column 1 alpha a_right (both rows)."""
    t = np.zeros((2, 2, 4), np.uint8)
    t[:, 0, 3] = a_left
    t[:, 1, 3] = a_right
    return t


def test_x3_fires_on_a_deciding_texel_line():
    # s = u = 0.5 -> s*W = 1: the line between column 0 (opaque) and 1 (clear)
    assert _flags(_scene(UNIT, _columns(255, 0)), _ray(0.5, 0.25),
                  isect=oracle.ALPHA_TEX) & oracle.X3


def test_x3_fires_on_a_row_line():
    t = np.zeros((2, 2, 4), np.uint8)
    t[0, :, 3] = 255   # row 0 opaque, row 1 clear; t = v = 0.5 -> t*H = 1
    assert _flags(_scene(UNIT, t), _ray(0.25, 0.5 - 2**-23), isect=oracle.ALPHA_TEX) & oracle.X3


def test_x3_silent_when_both_texels_agree():
    assert not _flags(_scene(UNIT, _columns(255, 255)), _ray(0.5, 0.25),
                      isect=oracle.ALPHA_TEX) & oracle.X3
    # a8 = 3 and a8 = 200 both pass .01: same decision, no flag
    assert not _flags(_scene(UNIT, _columns(3, 200)), _ray(0.5, 0.25),
                      isect=oracle.ALPHA_TEX) & oracle.X3


def test_x3_silent_away_from_texel_lines():
    assert not _flags(_scene(UNIT, _columns(255, 0)), _ray(0.3, 0.25),
                      isect=oracle.ALPHA_TEX) & oracle.X3


def test_x3_only_for_the_texture_intersector():
    assert not _flags(_scene(UNIT, _columns(255, 0)), _ray(0.5, 0.25),
                      isect=oracle.DEFAULT) & oracle.X3


def test_x3_threshold_straddle():
    """a8 = 2 | a8 = 3 straddle .01 (P:313 inclusive): a deciding line."""
    assert _flags(_scene(UNIT, _columns(2, 3)), _ray(0.5, 0.25),
                  isect=oracle.ALPHA_TEX) & oracle.X3


# ---- X4 checker edge -------------------------------------------------------------------
@pytest.mark.parametrize("x,y", [(0.25, 0.3), (0.3, 0.375), (0.125, 0.5)])
def test_x4_fires_when_u_or_v_times_m_is_integer(x, y):
    assert _flags(_scene(UNIT), _ray(x, y), isect=oracle.ALPHA_PROC, M=8) & oracle.X4


@pytest.mark.parametrize("x,y", [(0.3, 0.3), (0.26, 0.33)])
def test_x4_silent_inside_a_cell(x, y):
    assert not _flags(_scene(UNIT), _ray(x, y), isect=oracle.ALPHA_PROC, M=8) & oracle.X4


def test_x4_uses_the_call_frequency():
    # u*3 = 1 at u = 1/3 is a cell edge for M = 3 but not for M = 8 (8/3 = 2.67)
    x = np.float32(1.0) / np.float32(3.0)
    assert _flags(_scene(UNIT), _ray(float(x), 0.2), isect=oracle.ALPHA_PROC, M=3) & oracle.X4
    assert not _flags(_scene(UNIT), _ray(float(x), 0.2), isect=oracle.ALPHA_PROC, M=8) & oracle.X4


# ---- X5 bilinear alpha at the threshold ---------------------------------------------
# columns alpha 0 | 1: along s the bilinear alpha is 2s - 0.5 on [0.25, 0.75]
# (texel centres at s = .25 and .75), exact in fp32 for dyadic s
RAMP = _columns(0, 255)


@pytest.mark.parametrize("ds", [0.0, 2.0**-22, -(2.0**-22)])
def test_x5_fires_within_1e_6_of_the_threshold(ds):
    s = 0.5 + ds           # alpha = 0.5 + 2 ds: |alpha - thr| <= 4.8e-7 < 1e-6
    assert _flags(_scene(UNIT, RAMP), _ray(s, 0.25), isect=oracle.ALPHA_TEX_BILINEAR,
                  thr=0.5) & oracle.X5


@pytest.mark.parametrize("ds", [2.0**-18, -(2.0**-18), 0.1])
def test_x5_silent_outside_the_band(ds):
    s = 0.5 + ds           # |alpha - thr| >= 7.6e-6: the floor does not reach it
    assert not _flags(_scene(UNIT, RAMP), _ray(s, 0.25), isect=oracle.ALPHA_TEX_BILINEAR,
                      thr=0.5) & oracle.X5


def test_x5_exact_ramp_values():
    """The ramp itself (so the flag tests above sit where they claim): alpha(s) = 2s - .5."""
    for s, keep in ((0.5, True), (0.5 - 2.0**-22, False), (0.5 + 2.0**-22, True)):
        h = oracle.trace(_scene(UNIT, RAMP), _ray(s, 0.25), oracle.CLOSEST,
                         oracle.ALPHA_TEX_BILINEAR, alpha_threshold=0.5, nthreads=1)
        assert (h["prim"][0] == 0) == keep, s


def test_x5_not_for_nearest_rgba8():
    """Reading A7: no RGBA8 texel lies within 1e-6 of .01, so nearest lookups never set X5."""
    t = np.zeros((2, 2, 4), np.uint8)
    t[..., 3] = np.array([[2, 3], [3, 2]], np.uint8)
    rng = np.random.default_rng(0)
    xy = rng.uniform(0.01, 0.49, size=(256, 2))
    rays = np.concatenate([_ray(x, y) for x, y in xy])
    _, fl = oracle.trace(_scene(UNIT, t), rays, oracle.CLOSEST, oracle.ALPHA_TEX, flags=True,
                         nthreads=1)
    assert not np.any(fl & oracle.X5)


def test_x5_band_propagates_texcoord_error():
    """Non-dyadic geometry: the fp32 texcoords deviate from the double ones, and the band
    grows with W*|ds| — yet it stays far below the 1e-4 of round 1 for W = 2 (a band that
    flagged every ray would hide mismatches)."""
    tri = [0.1, 0.2, 0.0, 1.3, 0.1, 0.1, 0.2, 1.1, -0.1]
    rng = np.random.default_rng(3)
    rays = np.concatenate([_ray(x, y) for x, y in rng.uniform(0.2, 0.6, size=(512, 2))])
    _, fl = oracle.trace(_scene(tri, RAMP), rays, oracle.CLOSEST, oracle.ALPHA_TEX_BILINEAR,
                         alpha_threshold=0.5, flags=True, nthreads=1)
    assert (fl & oracle.X5).sum() <= 2   # |alpha - .5| < ~1e-6 has probability ~1e-5 per ray


def _double_bilinear_decision(tri, tex, thr, rays):
    """Independent float64 evaluation (numpy): MT on the same fp32 inputs, the lerp of
    the texcoords (0,0),(1,0),(0,1) and the bilinear alpha of SURVEY A.3 / reading A28."""
    v0, v1, v2 = (np.asarray(tri[i:i + 3], np.float64) for i in (0, 3, 6))
    o, d = rays[:, 0:3].astype(np.float64), rays[:, 4:7].astype(np.float64)
    e1, e2 = v1 - v0, v2 - v0
    p = np.cross(d, e2)
    det = p @ e1
    s = o - v0
    u = (s @ p) / det if np.ndim(det) == 0 else np.einsum("ij,ij->i", s, p) / det
    q = np.cross(s, e1)
    v = np.einsum("ij,ij->i", d, q) / det
    ss, tt = u, v                                     # texcoords (0,0), (1,0), (0,1)
    h, w = tex.shape[:2]
    a = tex[..., 3].astype(np.float64) / 255.0
    x, y = ss * w - 0.5, tt * h - 0.5
    x0, y0 = np.floor(x), np.floor(y)
    fx, fy = x - x0, y - y0
    i0, i1 = x0.astype(np.int64) % w, (x0.astype(np.int64) + 1) % w
    j0, j1 = y0.astype(np.int64) % h, (y0.astype(np.int64) + 1) % h
    al = ((1 - fx) * a[j0, i0] + fx * a[j0, i1]) * (1 - fy) + ((1 - fx) * a[j1, i0] + fx * a[j1, i1]) * fy
    return al >= thr, np.minimum(np.minimum(u, v), 1 - u - v)


def test_x5_covers_every_fp32_vs_fp64_disagreement():
    """Soundness of the X5 band: on a wide, steep texture (1024 columns alternating
    alpha 0 / 1, so |d alpha / d s| reaches W) the fp32 texcoords' rounding flips real
    decisions; every ray whose fp32 decision differs from the float64 one must be flagged
    X5, and such rays must exist (else the test proves nothing)."""
    tex = np.zeros((4, 1024, 4), np.uint8)
    tex[:, 1::2, 3] = 255
    tri = [0.1, 0.2, 0.0, 1.3, 0.1, 0.1, 0.2, 1.1, -0.1]
    rng = np.random.default_rng(11)
    n = 200_000
    xy = rng.uniform(0.25, 0.6, size=(n, 2))
    rays = np.zeros((n, 8), np.float32)
    rays[:, 0:2] = xy
    rays[:, 2] = -1.0
    rays[:, 3] = 1e-4
    rays[:, 6] = 1.0
    rays[:, 7] = np.inf
    h, fl = oracle.trace(_scene(tri, tex), rays, oracle.CLOSEST, oracle.ALPHA_TEX_BILINEAR,
                         alpha_threshold=0.5, flags=True)
    keep64, margin = _double_bilinear_decision(tri, tex, 0.5, rays)
    inside = margin > 1e-4                           # geometric hit certain on both sides
    keep32 = h["prim"] == 0
    differ = inside & (keep32 != keep64)
    assert differ.sum() >= 3, "no fp32/fp64 disagreement generated"
    assert np.all(fl[differ] & oracle.X5), np.nonzero(differ & ((fl & oracle.X5) == 0))[0][:5]
    # and the band stays a small class, not a blanket exclusion
    assert (fl[inside] & oracle.X5).astype(bool).mean() < 0.01


def test_eval_pairs_equals_eval_pair():
    """The batch form used by the parity checks is the per-pair function, element by element."""
    sc = W.random_soup(60, seed=9)
    rays = W.random_rays(300, seed=9).data
    prims = np.random.default_rng(9).integers(0, 60, 300)
    for isect in (oracle.DEFAULT, oracle.ALPHA_TEX, oracle.ALPHA_PROC):
        acc, h = oracle.eval_pairs(sc, rays, prims, isect)
        for i in range(0, 300, 7):
            a, t, u, v = oracle.eval_pair(sc, rays[i], int(prims[i]), isect)
            assert a == acc[i] and (t, u, v) == (h["t"][i], h["u"][i], h["v"][i])
    with pytest.raises(ValueError):
        oracle.eval_pairs(sc, rays[:1], [60])
