"""Two-level instancing ("object instancing, where the BVH will store
BVHs as primitives"; reading A27) — CPU only.

Pins of the oracle side (the ray map, brute force over instances, walker C) against
closed forms and the plain single-level oracle, then the product's host-only top-level
build checked structurally and by walker C == brute force.  No kernel is launched."""
import math

import numpy as np
import pytest

import workloads as W
from tests import bvh_check

MISS = 0xFFFFFFFF
INF = float("inf")


@pytest.fixture(scope="module")
def vsr():
    from paper_1912_12786_b200 import _build
    _build.build()
    from paper_1912_12786_b200 import vsr as V
    return V


def identity():
    return np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0], np.float32)


def dyadic_soup(n, seed, extent=6.0):
    """random_soup with vertices rounded to multiples of 1/64: every translation by a
    multiple of 1/64 below 2^10 is exact in fp32."""
    sc = W.random_soup(n, seed=seed, extent=extent)
    sc.vertices = (np.round(sc.vertices * 64.0) / 64.0).astype(np.float32)
    return sc


def dyadic_rays(n, seed):
    r = W.random_rays(n, seed=seed, extent=9.0, target=5.0).data.copy()
    r[:, 0:3] = np.round(r[:, 0:3] * 64.0) / 64.0
    return r


def random_affine(k, seed, extent=20.0):
    rng = np.random.default_rng(seed)
    m = W.object_from_world(rng.uniform(0, 2 * math.pi, k), rng.uniform(0.5, 2.0, k),
                            rng.uniform(-extent, extent, k), rng.uniform(-3, 3, k),
                            rng.uniform(-extent, extent, k), rng.uniform(-0.3, 0.3, k))
    # a non-uniform scale on some instances (A rows scaled independently)
    m = m.reshape(-1, 3, 4)
    m[::3, 1, :3] *= np.float32(0.5)
    return m.reshape(-1, 12)


# --------------------------------------------------------------------------- ray map pins

def test_ray_map_closed_forms(oracle_lib):
    o = oracle_lib
    rays = dyadic_rays(200, 1)
    assert np.array_equal(o.rays_to_object(rays, identity()), rays)
    t = identity()
    t[[3, 7, 11]] = [8.0, -4.25, 16.5]
    moved = o.rays_to_object(rays, t)
    assert np.array_equal(moved[:, 0:3], rays[:, 0:3] + np.float32([8.0, -4.25, 16.5]))
    assert np.array_equal(moved[:, 4:8], rays[:, 4:8]) and np.array_equal(moved[:, 3], rays[:, 3])
    # axis permutation with a sign: (x, y, z) -> (z, -x, y), exact
    p = np.array([0, 0, 1, 0, -1, 0, 0, 0, 0, 1, 0, 0], np.float32)
    q = o.rays_to_object(rays, p)
    assert np.array_equal(q[:, 0], rays[:, 2]) and np.array_equal(q[:, 1], -rays[:, 0])
    assert np.array_equal(q[:, 6], rays[:, 5]) and np.array_equal(q[:, 5], -rays[:, 4])


def test_ray_map_c_equals_numpy(oracle_lib):
    """walker.c's map and the brute force's numpy map are one reading, two codes."""
    o = oracle_lib
    rays = W.random_rays(300, seed=2).data
    for m in random_affine(8, 3):
        ref = o.rays_to_object(rays, m)
        for i in range(0, 300, 37):
            assert np.array_equal(o.ray_to_object(m, rays[i]), ref[i])


# --------------------------------------------------------------------------- brute force pins

def test_identity_instance_is_the_plain_scene(oracle_lib):
    o = oracle_lib
    sc = W.random_soup(300, seed=5)
    rays = W.random_rays(3000, seed=6)
    for q in (o.CLOSEST, o.ANY):
        for isect in (o.DEFAULT, o.ALPHA_TEX, o.ALPHA_PROC):
            ref = o.trace(sc, rays, q, isect)
            h, inst, fl, nt = o.trace_instances([sc], [0], [identity()], rays, q, isect)
            assert np.array_equal(h, ref)
            assert np.array_equal(inst, np.where(ref["prim"] != MISS, 0, MISS).astype(np.uint32))


def test_translated_instance_equals_moved_geometry(oracle_lib):
    """A = I, b = -c with dyadic c: the object-space MT is the world MT on geometry moved
    by +c, bit for bit (every subtraction is exact)."""
    o = oracle_lib
    sc = dyadic_soup(300, 7)
    rays = dyadic_rays(3000, 8)
    c = np.float32([3.5, -2.0, 1.25])
    m = identity()
    m[[3, 7, 11]] = -c
    moved = W.Scene("moved", (sc.vertices.reshape(-1, 3, 3) + c).reshape(-1, 9).astype(np.float32),
                    sc.geom_ids, sc.texcoords, sc.geom_texture, sc.textures)
    for isect in (o.DEFAULT, o.ALPHA_TEX):
        ref = o.trace(moved, rays, o.CLOSEST, isect)
        h, inst, _, _ = o.trace_instances([sc], [0], [m], rays, o.CLOSEST, isect)
        assert (ref["prim"] != MISS).sum() > 100
        assert np.array_equal(h, ref)


def test_two_instances_equal_the_concatenated_scene(oracle_lib):
    o = oracle_lib
    sc = dyadic_soup(200, 9)
    rays = dyadic_rays(4000, 10)
    cs = [np.float32([0, 0, 0]), np.float32([2.5, 0.5, -1.0])]
    ms, parts = [], []
    for c in cs:
        m = identity()
        m[[3, 7, 11]] = -c
        ms.append(m)
        parts.append(W.Scene("p", (sc.vertices.reshape(-1, 3, 3) + c).reshape(-1, 9).astype(np.float32),
                             sc.geom_ids, sc.texcoords, sc.geom_texture, sc.textures))
    cat, offs = W.concat_scenes(parts)
    ref, nt = o.trace(cat, rays, o.CLOSEST, o.ALPHA_TEX, ties=True)
    h, inst, fl, nti = o.trace_instances([sc], [0, 0], ms, rays, o.CLOSEST, o.ALPHA_TEX)
    hit = ref["prim"] != MISS
    assert np.array_equal(h["prim"] != MISS, hit)
    assert np.array_equal(h["t"], ref["t"])
    glob = np.where(hit, offs[np.minimum(inst, 1)] + h["prim"], MISS)
    ok = nt <= 1
    assert np.array_equal(glob[ok], ref["prim"][ok])


def test_instance_order_invariance(oracle_lib):
    o = oracle_lib
    models = [W.random_soup(150, seed=s, extent=3.0) for s in (11, 12)]
    rays = W.random_rays(3000, seed=13, extent=25.0, target=12.0)
    m = random_affine(12, 14, extent=10.0)
    bvh = np.arange(12) % 2
    h, inst, fl, nt = o.trace_instances(models, bvh, m, rays, o.CLOSEST, o.ALPHA_TEX)
    perm = np.random.default_rng(15).permutation(12)
    h2, inst2, fl2, nt2 = o.trace_instances(models, bvh[perm], m[perm], rays, o.CLOSEST, o.ALPHA_TEX)
    ok = (nt <= 1) & ((fl & o.X1) == 0)
    assert (h["prim"] != MISS).sum() > 200
    assert np.array_equal(h["t"], h2["t"])
    assert np.array_equal(h[ok], h2[ok])
    hit = (h["prim"] != MISS) & ok
    assert np.array_equal(inst[hit], perm[inst2[hit]])


# --------------------------------------------------------------------------- product top level

def _host_instances(vsr, models, bvh, m, max_leaf=1):
    scenes = [vsr.Scene.from_workload(s, device=-1).build() for s in models]
    inst = vsr.Instances(scenes, bvh, m, max_leaf_size=max_leaf)
    return scenes, inst


def _check_top(top, models_export, m, max_leaf):
    """Tree shape, every record in one leaf, nested boxes, and each instance's world
    image of its scene's root box (fp64) inside its leaf box."""
    nodes = top["nodes"]
    recs = top["records"]
    nf = nodes.view(np.float32)
    seen = np.zeros(recs.shape[0], np.int64)
    rf = recs.view(np.float32)

    def box_of(n, c):
        return (np.array([nf[n, 0 + c], nf[n, 4 + c], nf[n, 8 + c]]),
                np.array([nf[n, 2 + c], nf[n, 6 + c], nf[n, 10 + c]]))

    def visit(ref, lo, hi, depth):
        assert depth <= 64
        if ref & 0x80000000:
            first, cnt = ref & 0x03FFFFFF, ((ref >> 26) & 31) + 1
            assert cnt <= max_leaf
            for k in range(first, first + cnt):
                seen[k] += 1
                b = int(recs[k, 12])
                A = rf[k, :12].astype(np.float64).reshape(3, 4)
                inv = np.linalg.inv(A[:, :3])
                e = models_export[b]
                for c in range(8):
                    p = np.array([(e["root_hi"] if c & (1 << a) else e["root_lo"])[a] for a in range(3)],
                                 np.float64)
                    w = inv @ (p - A[:, 3])
                    assert np.all(w >= lo) and np.all(w <= hi)
            return
        for c in (0, 1):
            clo, chi = box_of(ref, c)
            assert np.all(clo >= lo) and np.all(chi <= hi)
            visit(int(nodes[ref, 12 + c]), clo, chi, depth + 1)

    visit(top["root_ref"], top["root_lo"].astype(np.float64), top["root_hi"].astype(np.float64), 0)
    assert np.all(seen == 1)
    assert sorted(recs[:, 13].tolist()) == list(range(recs.shape[0]))
    for k in range(recs.shape[0]):   # records carry the caller's matrix and bvh
        j = int(recs[k, 13])
        assert np.array_equal(rf[k, :12], m[j])


@pytest.mark.parametrize("max_leaf", [1, 3])
def test_product_top_level_valid(vsr, max_leaf):
    models = [W.random_soup(100, seed=s, extent=3.0) for s in (21, 22, 23)]
    m = random_affine(40, 24)
    bvh = np.random.default_rng(25).integers(0, 3, 40)
    scenes, inst = _host_instances(vsr, models, bvh, m, max_leaf)
    top = inst.export()
    assert top["records"].shape[0] == 40
    _check_top(top, [s.export() for s in scenes], m, max_leaf)


@pytest.mark.parametrize("max_leaf", [1, 2])
def test_walker_on_product_top_level_equals_bruteforce(vsr, oracle_lib, max_leaf):
    o = oracle_lib
    models = [W.random_soup(120, seed=s, extent=3.0) for s in (31, 32)]
    m = random_affine(30, 33, extent=12.0)
    bvh = np.arange(30) % 2
    rays = W.random_rays(4000, seed=34, extent=30.0, target=12.0)
    scenes, inst = _host_instances(vsr, models, bvh, m, max_leaf)
    top = inst.export()
    bottoms = [bvh_check.to_oracle(s.export()) for s in scenes]
    for isect in (o.DEFAULT, o.ALPHA_TEX, o.ALPHA_PROC):
        ref, rinst, fl, nt = o.trace_instances(models, bvh, m, rays, o.CLOSEST, isect)
        h, winst, c = o.walk_instances(top, top["records"], bottoms, rays, o.CLOSEST, isect)
        hit = ref["prim"] != MISS
        assert hit.sum() > 200
        assert np.array_equal(h["prim"] != MISS, hit)
        ok = hit & (nt <= 1) & ((fl & o.X1) == 0)
        assert np.array_equal(h["t"][hit], ref["t"][hit])
        assert np.array_equal(h[ok], ref[ok])
        assert np.array_equal(winst[ok], rinst[ok])
        assert np.all(winst[~hit] == MISS)
        # any-hit: the returned (instance, prim) is accepted, with the oracle's (t, u, v)
        a, ainst, ac = o.walk_instances(top, top["records"], bottoms, rays, o.ANY, isect)
        assert np.array_equal(a["prim"] != MISS, hit)
        for i in np.nonzero(hit)[0][:300]:
            j = int(ainst[i])
            r = o.rays_to_object(rays.data[i:i + 1], m[j])[0]
            acc, t, u, v = o.eval_pair(models[bvh[j]], r, int(a["prim"][i]), isect)
            assert acc and (t, u, v) == (a["t"][i], a["u"][i], a["v"][i])
        assert np.all(ac["tris"] <= c["tris"])


def test_walker_instance_counts_closed_form(oracle_lib, vsr):
    """One instance of a single-leaf quad pair: root(top, leaf) 1 + bottom root 1 box tests
    and 2 triangle tests for a ray through it; 1 box test for a ray missing the top root."""
    o = oracle_lib
    q = W.stacked_quads(1, z0=1.0)
    scenes, inst = _host_instances(vsr, [q], [0], [identity()])
    top = inst.export()
    assert top["root_ref"] & 0x80000000    # one instance: the top root is a leaf
    bottoms = [bvh_check.to_oracle(scenes[0].export())]
    rays = np.array([[0.3, 0.6, 0, 1e-4, 0, 0, 1, INF],
                     [500, 500, 0, 1e-4, 0, 0, 1, INF]], np.float32)
    h, wi, c = o.walk_instances(top, top["records"], bottoms, rays, o.CLOSEST, o.COUNT)
    assert h["t"][0] == 1.0 and wi[0] == 0
    assert (c["boxes"][0], c["tris"][0]) == (2, 2)
    assert (c["boxes"][1], c["tris"][1]) == (1, 0) and wi[1] == MISS


def test_instances_validation(vsr):
    sc = vsr.Scene.from_workload(W.random_soup(50, seed=41), device=-1).build()
    bad = identity().copy()
    bad[5] = 0.0          # singular (row 1 of A is zero)
    with pytest.raises(vsr.VsrError):
        vsr.Instances([sc], [0], [bad])
    nan = identity().copy()
    nan[3] = np.nan
    with pytest.raises(vsr.VsrError):
        vsr.Instances([sc], [0], [nan])
    with pytest.raises(vsr.VsrError):
        vsr.Instances([sc], [1], [identity()])            # bvh index out of range
    unbuilt = vsr.Scene.from_workload(W.random_soup(50, seed=42), device=-1)
    with pytest.raises(vsr.VsrError):
        vsr.Instances([unbuilt], [0], [identity()])
    ok = vsr.Instances([sc], [0, 0], [identity(), identity()])
    assert ok.export()["records"].shape[0] == 2
    import ctypes as C
    h = np.zeros((1, 4), np.float32)
    r = np.zeros((1, 8), np.float32)
    st = vsr.lib().vsr_trace_instances(ok._h, r.ctypes.data, 1, 0, 1, None, h.ctypes.data, None,
                                       None, None)
    assert st == vsr.ERR_UNSUPPORTED     # host-only instances are not traceable
    del C


def test_instances_multi_walker(vsr, oracle_lib):
    """Multi-hit over instances: k = 1 is the closest query; for k = 4 the kept t lists equal the
    k smallest accepted t over all instances by brute force."""
    o = oracle_lib
    models = [W.random_soup(120, seed=s, extent=3.0) for s in (51, 52)]
    m = random_affine(24, 53, extent=12.0)
    bvh = np.arange(24) % 2
    rays = W.random_rays(2000, seed=54, extent=30.0, target=12.0)
    scenes, inst = _host_instances(vsr, models, bvh, m)
    top = inst.export()
    bottoms = [bvh_check.to_oracle(s.export()) for s in scenes]
    h1, n1, i1, c1 = o.walk_instances_multi(top, top["records"], bottoms, rays, 1, o.ALPHA_TEX)
    hc, ic, cc = o.walk_instances(top, top["records"], bottoms, rays, o.CLOSEST, o.ALPHA_TEX)
    assert np.array_equal(h1[:, 0], hc) and np.array_equal(i1[:, 0], ic) and np.array_equal(c1, cc)
    k = 4
    h, nh, ii, c = o.walk_instances_multi(top, top["records"], bottoms, rays, k, o.ALPHA_TEX)
    all_t = []
    for j in range(len(bvh)):
        hm, nm, _ = o.trace_multi(models[bvh[j]], o.rays_to_object(rays, m[j]), k, o.ALPHA_TEX)
        all_t.append(np.where(hm["prim"] != MISS, hm["t"], np.inf))
    best = np.sort(np.concatenate(all_t, axis=1), axis=1)[:, :k]
    assert np.array_equal(np.where(h["prim"] != MISS, h["t"], np.inf), best.astype(np.float32))
    assert np.array_equal(nh, (best < np.inf).sum(axis=1))
    assert np.all(ii[h["prim"] == MISS] == MISS)
    # every kept (instance, prim) is an accepted pair with exactly the kept (t, u, v)
    for i in range(0, rays.n, 7):
        for j in range(int(nh[i])):
            q = int(ii[i, j])
            ro = o.rays_to_object(rays.data[i:i + 1], m[q])[0]
            acc, t, u, v = o.eval_pair(models[bvh[q]], ro, int(h["prim"][i, j]), o.ALPHA_TEX)
            assert acc and (t, u, v) == (h["t"][i, j], h["u"][i, j], h["v"][i, j])


def _aimed_rays(targets, dist, n, seed):
    """n rays from origins `dist` away (random directions) through random target points."""
    rng = np.random.default_rng(seed)
    p = targets[rng.integers(0, targets.shape[0], n)] + rng.uniform(-2.0, 2.0, (n, 3))
    u = rng.normal(size=(n, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    o = p + dist * u
    r = np.zeros((n, 8), np.float32)
    r[:, 0:3] = o
    r[:, 3] = 1e-4
    r[:, 4:7] = (p - o) * rng.uniform(0.5, 2.0, (n, 1))
    r[:, 7] = np.inf
    return r


@pytest.mark.parametrize("dist", [3e2, 1e5])
def test_instances_conservative_at_any_distance(vsr, oracle_lib, dist):
    """Reading A27, round 2: the instance world boxes are proven conservative only for ray
    origins with max |o_k| <= r_safe (exported); beyond it the walk visits every instance.
    At 10^4 model diagonals (origin 1e5 away, model diagonal ~10) the walker over the
    product's top level must equal brute force over all instances, as it does near by."""
    o = oracle_lib
    models = [W.random_soup(120, seed=s, extent=3.0) for s in (51, 52)]
    m = random_affine(30, 53, extent=12.0)
    bvh = np.arange(30) % 2
    scenes, inst = _host_instances(vsr, models, bvh, m, 1)
    top = inst.export()
    assert 100.0 < top["r_safe"] < 1e5      # non-trivial, and exceeded by the far rays
    bottoms = [bvh_check.to_oracle(s.export()) for s in scenes]
    centres = -np.einsum("kij,kj->ki", np.linalg.inv(m.reshape(-1, 3, 4)[:, :, :3].astype(np.float64)),
                         m.reshape(-1, 3, 4)[:, :, 3].astype(np.float64))
    rays = _aimed_rays(centres, dist, 1500, int(dist))
    far = np.abs(rays[:, 0:3]).max(axis=1) > top["r_safe"]
    assert far.all() if dist > 1e4 else not far.any()
    ref, rinst, fl, nt = o.trace_instances(models, bvh, m, rays, o.CLOSEST, o.DEFAULT)
    h, winst, c = o.walk_instances(top, top["records"], bottoms, rays, o.CLOSEST, o.DEFAULT)
    hit = ref["prim"] != MISS
    assert hit.sum() > 100
    assert np.array_equal(h["prim"] != MISS, hit)
    assert np.array_equal(h["t"][hit], ref["t"][hit])
    if dist > 1e4:   # the linear path: the top root box (1) + every instance's root box
        assert np.all(c["boxes"] >= 1 + 30)
