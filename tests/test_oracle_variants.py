"""Pins for the NEXT-4 sampling variants (reading A28):
bilinear alpha and the texcoord-space procedural checker — CPU only.

Bilinear tex2D is pinned to closed forms (texel centres reduce to the nearest lookup
exactly; edge midpoints and the wrap seam are the mean of two texels; a constant texture is
that constant) and to the definition evaluated in fp64; the checker on texcoords reduces to
the barycentric checker when the texcoords are the barycentric frame."""
import numpy as np
import pytest

import workloads as W

MISS = 0xFFFFFFFF


def tex(w, h, seed):
    t = np.random.default_rng(seed).integers(0, 256, (h, w, 4)).astype(np.uint8)
    return t


def test_bilinear_at_texel_centres_is_nearest(oracle_lib):
    o = oracle_lib
    t = tex(8, 4, 1)
    for j in range(4):
        for i in range(8):
            s, tt = np.float32((i + 0.5) / 8), np.float32((j + 0.5) / 4)
            assert o.tex_alpha_bilinear(t, s, tt) == o.tex_alpha(t, s, tt) == np.float32(t[j, i, 3]) / np.float32(255)


def test_bilinear_midpoints_and_wrap_seam(oracle_lib):
    o = oracle_lib
    t = tex(8, 4, 2)
    a = t[..., 3].astype(np.float64) / 255.0
    for j in range(4):
        for i in range(8):
            s, tt = np.float32((i + 1.0) / 8), np.float32((j + 0.5) / 4)   # between i and i+1
            want = 0.5 * (a[j, i] + a[j, (i + 1) % 8])
            assert abs(o.tex_alpha_bilinear(t, s, tt) - want) < 2e-7
    # s = 0 sits halfway between the last and the first column (wrap)
    for j in range(4):
        want = 0.5 * (a[j, 7] + a[j, 0])
        assert abs(o.tex_alpha_bilinear(t, np.float32(0.0), np.float32((j + 0.5) / 4)) - want) < 2e-7
    # t = 1 + 0.5/H wraps onto row 0
    assert o.tex_alpha_bilinear(t, np.float32(0.5 / 8), np.float32(1.0 + 0.5 / 4)) == np.float32(t[0, 0, 3]) / np.float32(255)


def test_bilinear_constant_texture(oracle_lib):
    o = oracle_lib
    t = np.full((5, 7, 4), 77, np.uint8)
    rng = np.random.default_rng(3)
    for s, tt in rng.uniform(-3, 3, (200, 2)).astype(np.float32):
        assert abs(o.tex_alpha_bilinear(t, s, tt) - 77 / 255) < 3e-7


def test_bilinear_matches_fp64_definition(oracle_lib):
    """The textbook bilinear filter (texel centres at (i+.5)/W, wrap) in fp64, vectorised
    differently from the C oracle (corner weights, not nested lerps)."""
    o = oracle_lib
    t = tex(13, 9, 4)
    a = t[..., 3].astype(np.float64) / 255.0
    rng = np.random.default_rng(5)
    st = rng.uniform(-2, 3, (2000, 2)).astype(np.float32)
    x = st[:, 0].astype(np.float64) * 13 - 0.5
    y = st[:, 1].astype(np.float64) * 9 - 0.5
    i0, j0 = np.floor(x).astype(np.int64), np.floor(y).astype(np.int64)
    fx, fy = x - i0, y - j0
    want = (a[j0 % 9, i0 % 13] * (1 - fx) * (1 - fy) + a[j0 % 9, (i0 + 1) % 13] * fx * (1 - fy)
            + a[(j0 + 1) % 9, i0 % 13] * (1 - fx) * fy + a[(j0 + 1) % 9, (i0 + 1) % 13] * fx * fy)
    got = np.array([o.tex_alpha_bilinear(t, s, u) for s, u in st])
    assert np.max(np.abs(got - want)) < 5e-6


def test_uv_checker_reduces_to_barycentric_checker(oracle_lib):
    """texcoords (0,0), (1,0), (0,1): (s, t) == (u, v) exactly, so the two checkers agree."""
    o = oracle_lib
    sc = W.random_soup(400, seed=6)
    sc.texcoords = np.tile(np.array([0, 0, 1, 0, 0, 1], np.float32), (sc.num_tris, 1))
    rays = W.random_rays(3000, seed=7)
    for q in (o.CLOSEST, o.ANY):
        a = o.trace(sc, rays, q, o.ALPHA_PROC, checker_freq=5)
        b = o.trace(sc, rays, q, o.ALPHA_PROC_UV, checker_freq=5)
        assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", ["ALPHA_TEX_BILINEAR", "ALPHA_PROC_UV"])
def test_variant_walker_equals_bruteforce(oracle_lib, kind):
    o = oracle_lib
    k = getattr(o, kind)
    sc = W.random_soup(800, seed=8, size=2.0)
    rays = W.random_rays(4000, seed=9)
    b = o.build_bvh(sc, 2)
    thr = 0.5    # the soup's alpha is uniform on [0, 1]: about half of the geometric hits pass
    ref, fl, nt = o.trace(sc, rays, o.CLOSEST, k, alpha_threshold=thr, flags=True, ties=True)
    h, c = o.walk(b, rays, o.CLOSEST, k, alpha_threshold=thr)
    hit = ref["prim"] != MISS
    assert 200 < hit.sum() < len(hit)
    assert np.array_equal(h["prim"] != MISS, hit)
    ok = (nt <= 1) & (fl == 0)
    assert np.array_equal(h[ok], ref[ok])
    # the variant vetoes some geometric hits the default keeps
    d = o.trace(sc, rays, o.CLOSEST, o.DEFAULT)
    assert (d["prim"] != ref["prim"]).sum() > 50
