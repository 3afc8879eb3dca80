"""GPU parity of the NEXT-4 sampling variants (ALPHA_TEXTURE_BILINEAR, ALPHA_PROCEDURAL_UV;
DESIGN.md reading A28): bit-exact vs walker C on the exported BVH (fp32 in the same order on
both sides, so every filter decision matches), and vs the brute force outside its ambiguity
flags; also through the multi-hit, list and pinhole entry points."""
import numpy as np
import pytest

import workloads as W
from tests import bvh_check

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


def kinds(V, o):
    return ((V.ALPHA_TEXTURE_BILINEAR, o.ALPHA_TEX_BILINEAR), (V.ALPHA_PROCEDURAL_UV, o.ALPHA_PROC_UV))


def run(V, scene, rays, q, k, thr):
    r = torch.from_numpy(np.ascontiguousarray(rays, np.float32)).cuda()
    h, _ = scene.trace(r, q, k, alpha_threshold=thr, checker_freq=5)
    torch.cuda.synchronize()
    return V.hits_to_numpy(h)


@pytest.mark.parametrize("thr", [0.01, 0.5])
def test_variants_soup(V, oracle_lib, thr):
    o = oracle_lib
    sc = W.random_soup(2000, seed=80, size=2.0)
    rays = W.random_rays(6001, seed=81).data
    scene = V.Scene.from_workload(sc).build()
    b = bvh_check.to_oracle(scene.export())
    for k, ok in kinds(V, o):
        for q, oq in ((V.CLOSEST, o.CLOSEST), (V.ANY, o.ANY)):
            h = run(V, scene, rays, q, k, thr)
            wh, _ = o.walk(b, rays, oq, ok, alpha_threshold=thr, checker_freq=5)
            assert np.array_equal(h.view(np.uint32), wh.view(np.uint32)), (k, q, thr)
        ref, fl, nt = o.trace(sc, rays, o.CLOSEST, ok, alpha_threshold=thr, checker_freq=5,
                              flags=True, ties=True)
        h = run(V, scene, rays, V.CLOSEST, k, thr)
        good = (fl == 0) & (nt <= 1)
        assert good.mean() > 0.95
        assert np.array_equal(h[good], ref[good])


def test_variants_c1_and_forest(V, oracle_lib):
    o = oracle_lib
    for name, res in (("C1", None), ("C2", (480, 272))):
        sc, rays = W.config(name, *(res or (None, None)))
        scene = V.Scene.from_workload(sc).build()
        b = bvh_check.to_oracle(scene.export())
        for k, ok in kinds(V, o):
            for q, oq in ((V.CLOSEST, o.CLOSEST), (V.ANY, o.ANY)):
                h = run(V, scene, rays.data, q, k, 0.3)
                wh, _ = o.walk(b, rays.data, oq, ok, alpha_threshold=0.3, checker_freq=5)
                assert np.array_equal(h.view(np.uint32), wh.view(np.uint32)), (name, k, q)


def test_variants_multi_list_pinhole(V, oracle_lib):
    o = oracle_lib
    sc = W.random_soup(1500, seed=82, size=2.0)
    rays = W.random_rays(3001, seed=83).data
    r = torch.from_numpy(rays).cuda()
    scene = V.Scene.from_workload(sc).build()
    b = bvh_check.to_oracle(scene.export())
    for k, ok in kinds(V, o):
        hm, nm, _ = scene.trace_multi(r, 4, k, alpha_threshold=0.5, checker_freq=5)
        torch.cuda.synchronize()
        wh, wn, _ = o.walk_multi(b, rays, 4, ok, alpha_threshold=0.5, checker_freq=5)
        assert np.array_equal(V.hits_to_numpy(hm.reshape(-1, 4)).view(np.uint32).reshape(-1, 4, 4),
                              wh.view(np.uint32).reshape(-1, 4, 4))
        subs = W.split_scene(sc, 3)
        parts = [V.Scene.from_workload(s).build() for s in subs]
        g = V.Group(parts)
        hg, wg, _ = g.trace(r, V.CLOSEST, k, alpha_threshold=0.5, checker_freq=5)
        torch.cuda.synchronize()
        lh, lw, _ = o.walk_list([bvh_check.to_oracle(p.export()) for p in parts], rays, o.CLOSEST,
                                ok, alpha_threshold=0.5, checker_freq=5)
        assert np.array_equal(V.hits_to_numpy(hg).view(np.uint32), lh.view(np.uint32))
    # pinhole (fused ray generation) with a variant equals the host-ray path
    sc2, rays2 = W.config("C2", 128, 64)
    s2 = V.Scene.from_workload(sc2).build()
    eye, look, up, fov, _, _, _ = W.CAMERAS["C2"]
    cam = V.pinhole_camera(eye, look, up, fov, 128, 64)
    for k, _ in kinds(V, o):
        h1, _ = s2.trace(torch.from_numpy(rays2.data).cuda(), V.CLOSEST, k, alpha_threshold=0.3)
        h2, _ = s2.trace_pinhole(cam, V.CLOSEST, k, alpha_threshold=0.3)
        torch.cuda.synchronize()
        assert torch.equal(h1.view(torch.int32), h2.view(torch.int32))
