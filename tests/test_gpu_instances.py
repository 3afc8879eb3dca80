"""GPU parity of two-level instancing through
vsr_trace_instances: hits, instance indices and counts bit-exact vs walker C on the
exported top level + bottoms; closest hits vs the brute force over all instances."""
import numpy as np
import pytest

import workloads as W
from tests import bvh_check
from tests.test_instances_cpu import random_affine

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


def run(V, inst, rays_np, q, k):
    r = torch.from_numpy(np.ascontiguousarray(rays_np, np.float32)).cuda()
    hits, ii, counts = inst.trace(r, q, k)
    torch.cuda.synchronize()
    return (V.hits_to_numpy(hits), ii.cpu().numpy().astype(np.uint32),
            V.counts_to_numpy(counts) if counts is not None else None)


KINDS = ("NONE", "DEFAULT", "ALPHA_TEXTURE", "ALPHA_PROCEDURAL", "COUNT", "COUNT_ALPHA_TEXTURE")


def setup(V, models, bvh, m, max_leaf=1):
    scenes = [V.Scene.from_workload(s).build() for s in models]
    inst = V.Instances(scenes, bvh, m, max_leaf_size=max_leaf)
    top = inst.export()
    bottoms = [bvh_check.to_oracle(s.export()) for s in scenes]
    return scenes, inst, top, bottoms


@pytest.mark.parametrize("max_leaf", [1, 3])
def test_instances_vs_walker_and_bruteforce(V, oracle_lib, max_leaf):
    o = oracle_lib
    models = [W.random_soup(150, seed=s, extent=3.0, size=1.5) for s in (51, 52, 53)]
    m = random_affine(48, 54, extent=12.0)
    bvh = np.arange(48) % 3
    rays = W.random_rays(6001, seed=55, extent=30.0, target=12.0).data   # ragged tail
    scenes, inst, top, bottoms = setup(V, models, bvh, m, max_leaf)
    for q, oq in ((V.CLOSEST, o.CLOSEST), (V.ANY, o.ANY)):
        for name in KINDS:
            k = getattr(V, name)
            ok = okind(V, o, k)
            h, ii, c = run(V, inst, rays, q, k)
            wh, wi, wc = o.walk_instances(top, top["records"], bottoms, rays, oq, ok)
            assert np.array_equal(h.view(np.uint32), wh.view(np.uint32)), (name, q)
            assert np.array_equal(ii, wi), (name, q)
            if c is not None:
                assert np.array_equal(c["boxes"], wc["boxes"]), (name, q)
                assert np.array_equal(c["tris"], wc["tris"]), (name, q)
                if k == V.COUNT_ALPHA_TEXTURE:
                    assert np.array_equal(c["alpha"], wc["alpha"])
            if q == V.CLOSEST and name in ("DEFAULT", "ALPHA_TEXTURE", "ALPHA_PROCEDURAL"):
                ref, rinst, fl, nt = o.trace_instances(models, bvh, m, rays, oq, ok)
                hit = ref["prim"] != MISS
                assert hit.sum() > 500
                assert np.array_equal(h["prim"] != MISS, hit)
                assert np.array_equal(h["t"][hit], ref["t"][hit])
                good = hit & (nt <= 1) & ((fl & o.X1) == 0)
                assert np.array_equal(h[good], ref[good])
                assert np.array_equal(ii[good], rinst[good])


def test_instanced_forest_frame(V, oracle_lib):
    """The NEXT-2 workload (instanced tree models over the C2 ground) at 480x272: GPU ==
    walker bit-exact for hits, instance ids and counts; closest hits on a ray sample vs the
    brute force over all instances."""
    o = oracle_lib
    models, bvh, m = W.instanced_forest(n_instances=2000, cards=32)
    rays = W.rays_for("C2", 480, 272).data
    scenes, inst, top, bottoms = setup(V, models, bvh, m)
    for q, oq in ((V.ANY, o.ANY), (V.CLOSEST, o.CLOSEST)):
        for k in (V.ALPHA_TEXTURE, V.COUNT_ALPHA_TEXTURE):
            h, ii, c = run(V, inst, rays, q, k)
            wh, wi, wc = o.walk_instances(top, top["records"], bottoms, rays, oq, okind(V, o, k))
            assert np.array_equal(h.view(np.uint32), wh.view(np.uint32))
            assert np.array_equal(ii, wi)
            if c is not None:
                assert np.array_equal(c["boxes"], wc["boxes"]) and np.array_equal(c["tris"], wc["tris"])
        assert (h["prim"] != MISS).mean() > 0.05
    sample = np.random.default_rng(3).choice(rays.shape[0], 1500, replace=False)
    h, ii, _ = run(V, inst, rays, V.CLOSEST, V.ALPHA_TEXTURE)
    ref, rinst, fl, nt = o.trace_instances(models, bvh, m, rays[sample], o.CLOSEST, o.ALPHA_TEX)
    hs = h[sample]
    hit = ref["prim"] != MISS
    assert np.array_equal(hs["prim"] != MISS, hit)
    good = hit & (nt <= 1) & ((fl & o.X1) == 0)
    assert np.array_equal(hs[good], ref[good]) and np.array_equal(ii[sample][good], rinst[good])


def test_instances_edge_cases(V, oracle_lib):
    o = oracle_lib
    models = [W.random_soup(60, seed=61, extent=2.0)]
    m = random_affine(5, 62, extent=4.0)
    scenes, inst, top, bottoms = setup(V, models, np.zeros(5, np.uint32), m)
    # n = 0 and a ray missing everything
    r0 = torch.zeros((0, 8), dtype=torch.float32, device="cuda")
    inst.trace(r0, V.CLOSEST, V.DEFAULT)
    far = np.array([[1e4, 1e4, 1e4, 1e-4, 1, 0, 0, np.inf]], np.float32)
    h, ii, c = run(V, inst, far, V.CLOSEST, V.COUNT)
    # a missing ray tests the top root only — unless its origin is beyond r_safe (reading
    # A27), where every instance's root box is tested too
    boxes = 1 + (5 if float(np.abs(far[0, :3]).max()) > top["r_safe"] else 0)
    assert h["prim"][0] == MISS and ii[0] == MISS and c["boxes"][0] == boxes and c["tris"][0] == 0
    # hits buffer only (no instance buffer)
    rays = W.random_rays(1000, seed=63, extent=10.0, target=4.0).data
    rt = torch.from_numpy(rays).cuda()
    hits = torch.empty((1000, 4), dtype=torch.float32, device="cuda")
    V._check(V.lib().vsr_trace_instances(inst._h, rt.data_ptr(), 1000, V.CLOSEST, V.DEFAULT, None,
                                         hits.data_ptr(), None, None, V._stream_handle(None)))
    torch.cuda.synchronize()
    wh, wi, wc = o.walk_instances(top, top["records"], bottoms, rays, o.CLOSEST, o.DEFAULT)
    assert np.array_equal(V.hits_to_numpy(hits).view(np.uint32), wh.view(np.uint32))
    # run-time controls are not provided for instanced queries
    with pytest.raises(V.VsrError):
        inst.trace(rt, V.CLOSEST, V.RUNTIME_SWITCH_DEFAULT)


@pytest.mark.parametrize("k", [1, 4])
def test_instances_multi_vs_walker(V, oracle_lib, k):
    o = oracle_lib
    models = [W.random_soup(150, seed=s, extent=3.0, size=1.5) for s in (71, 72)]
    m = random_affine(32, 73, extent=12.0)
    bvh = np.arange(32) % 2
    rays = W.random_rays(4001, seed=74, extent=30.0, target=12.0).data
    scenes, inst, top, bottoms = setup(V, models, bvh, m)
    r = torch.from_numpy(rays).cuda()
    for kind, ok in ((V.ALPHA_TEXTURE, o.ALPHA_TEX), (V.COUNT_ALPHA_TEXTURE, o.ALPHA_TEX)):
        h, n, ii, c = inst.trace_multi(r, k, kind)
        torch.cuda.synchronize()
        wh, wn, wi, wc = o.walk_instances_multi(top, top["records"], bottoms, rays, k, ok)
        assert np.array_equal(V.hits_to_numpy(h.reshape(-1, 4)).view(np.uint32),
                              wh.reshape(-1).view(np.uint32))
        assert np.array_equal(n.cpu().numpy().astype(np.uint32), wn)
        assert np.array_equal(ii.cpu().numpy().astype(np.uint32), wi)
        if c is not None:
            cc = V.counts_to_numpy(c)
            assert np.array_equal(cc["boxes"], wc["boxes"]) and np.array_equal(cc["tris"], wc["tris"])


def test_instanced_forest_full_frame_vs_walker(V, oracle_lib):
    """The NEXT-2 bench workload at full size (1080p, 10k instances): ANY + alpha texture as the
    bench times it, hits and instance ids bit-exact vs walker C on the whole frame."""
    o = oracle_lib
    models, bvh, m = W.instanced_forest()
    rays = W.rays_for("C2").data
    scenes, inst, top, bottoms = setup(V, models, bvh, m)
    h, ii, _ = run(V, inst, rays, V.ANY, V.ALPHA_TEXTURE)
    wh, wi, _ = o.walk_instances(top, top["records"], bottoms, rays, o.ANY, o.ALPHA_TEX)
    assert np.array_equal(h.view(np.uint32), wh.view(np.uint32))
    assert np.array_equal(ii, wi)
    assert (h["prim"] != MISS).mean() > 0.3


@pytest.mark.parametrize("dist", [3e2, 1e5])
def test_instances_far_origins(V, oracle_lib, dist):
    """Reading A27 (round 2): origins beyond the exported r_safe take the linear path over
    every instance; at 10^4 model diagonals the GPU equals walker C bit for bit (hits,
    instance ids, counts, both queries, multi-hit k = 4) and brute force on hit/miss and t."""
    from tests.test_instances_cpu import _aimed_rays
    o = oracle_lib
    models = [W.random_soup(120, seed=s, extent=3.0) for s in (51, 52)]
    m = random_affine(30, 53, extent=12.0)
    bvh = np.arange(30) % 2
    scenes, inst, top, bottoms = setup(V, models, bvh, m, 1)
    centres = -np.einsum("kij,kj->ki", np.linalg.inv(m.reshape(-1, 3, 4)[:, :, :3].astype(np.float64)),
                         m.reshape(-1, 3, 4)[:, :, 3].astype(np.float64))
    rays = _aimed_rays(centres, dist, 3001, int(dist) + 1)
    assert (np.abs(rays[:, 0:3]).max(axis=1) > top["r_safe"]).all() == (dist > 1e4)
    for q, oq in ((V.CLOSEST, o.CLOSEST), (V.ANY, o.ANY)):
        for name in ("DEFAULT", "COUNT", "ALPHA_TEXTURE"):
            k = getattr(V, name)
            h, ii, c = run(V, inst, rays, q, k)
            wh, wi, wc = o.walk_instances(top, top["records"], bottoms, rays, oq, okind(V, o, k))
            assert h.tobytes() == wh.tobytes() and np.array_equal(ii, wi), (name, q)
            if c is not None:
                assert np.array_equal(c["boxes"], wc["boxes"]) and np.array_equal(c["tris"], wc["tris"])
    ref, _, _, _ = o.trace_instances(models, bvh, m, rays, o.CLOSEST, o.DEFAULT)
    h, _, _ = run(V, inst, rays, V.CLOSEST, V.DEFAULT)
    hit = ref["prim"] != MISS
    assert hit.sum() > 100 and np.array_equal(h["prim"] != MISS, hit)
    assert np.array_equal(h["t"][hit], ref["t"][hit])
    r = torch.from_numpy(rays).cuda()
    mh, mn, mi, _ = inst.trace_multi(r, 4, V.DEFAULT)
    torch.cuda.synchronize()
    wh4, wn4, wi4, _ = o.walk_instances_multi(top, top["records"], bottoms, rays, 4, o.DEFAULT)
    assert V.hits_to_numpy(mh.reshape(-1, 4)).tobytes() == wh4.reshape(-1).tobytes()
    assert np.array_equal(mn.cpu().numpy().astype(np.uint32), wn4)
