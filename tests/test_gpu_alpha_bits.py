"""GPU parity of the 1-bit alpha plane: ALPHA_TEXTURE
reads a per-threshold plane of (a8 >= a_min) in 32×32-texel tiles when every texture's W and H
are multiples of 32, and the A8 plane otherwise. Both paths must give the walker C result bit
for bit, and each other's bytes, at every threshold — including ones that pass everything or
nothing — on textures that are non-square and not powers of two, and past the scene's cache of
eight planes."""
import numpy as np
import pytest

import workloads as W
from tests import bvh_check

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def V():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_12786_b200 import _build
    _build.build()
    from paper_1912_12786_b200 import vsr
    return vsr


def soup_with(shapes, seed):
    sc = W.random_soup(3000, seed=seed, size=2.0, n_geoms=6, n_textures=len(shapes))
    rng = np.random.default_rng(seed + 1)
    sc.textures = [rng.integers(0, 256, (h, w, 4)).astype(np.uint8) for (h, w) in shapes]
    return sc


def trace(V, s, rays, q, thr, monkeypatch, bits):
    monkeypatch.setenv("VSR_ALPHA_BITS", "1" if bits else "0")
    r = torch.from_numpy(np.ascontiguousarray(rays, np.float32)).cuda()
    h, _ = s.trace(r, q, V.ALPHA_TEXTURE, alpha_threshold=thr)
    torch.cuda.synchronize()
    return V.hits_to_numpy(h)


THRESHOLDS = [0.0, 1e-6, 0.01, 0.25, 0.5, 0.75, 0.999, 1.0, 1.5, 0.3, 0.6]   # > 8 distinct a_min


@pytest.mark.parametrize("shapes", [[(64, 96), (32, 160), (128, 128)],    # plane (32-aligned)
                                    [(64, 96), (24, 40)],                  # one unaligned: A8
                                    [(32, 32)]])
def test_bits_plane_equals_a8_and_walker(V, oracle_lib, monkeypatch, shapes):
    o = oracle_lib
    sc = soup_with(shapes, seed=90 + len(shapes))
    rays = W.random_rays(20011, seed=91).data
    s = V.Scene.from_workload(sc).build()
    b = bvh_check.to_oracle(s.export())
    for thr in THRESHOLDS:
        for q, oq in ((V.ANY, o.ANY), (V.CLOSEST, o.CLOSEST)):
            hb = trace(V, s, rays, q, thr, monkeypatch, True)
            ha = trace(V, s, rays, q, thr, monkeypatch, False)
            assert hb.tobytes() == ha.tobytes(), (shapes, thr, q)
            wh, _ = o.walk(b, rays, oq, o.ALPHA_TEX, alpha_threshold=thr)
            assert np.array_equal(hb.view(np.uint32), wh.view(np.uint32)), (shapes, thr, q)


def test_bits_plane_on_the_forest(V, oracle_lib, monkeypatch):
    """C2's 1024² textures (the headline path), a 480×272 frame, both queries."""
    o = oracle_lib
    sc, rays = W.config("C2", 480, 272)
    s = V.Scene.from_workload(sc).build()
    b = bvh_check.to_oracle(s.export())
    for thr in (0.01, 0.5):
        for q, oq in ((V.ANY, o.ANY), (V.CLOSEST, o.CLOSEST)):
            hb = trace(V, s, rays.data, q, thr, monkeypatch, True)
            ha = trace(V, s, rays.data, q, thr, monkeypatch, False)
            assert hb.tobytes() == ha.tobytes()
            wh, _ = o.walk(b, rays.data, oq, o.ALPHA_TEX, alpha_threshold=thr)
            assert np.array_equal(hb.view(np.uint32), wh.view(np.uint32)), (thr, q)


@pytest.mark.parametrize("k", [4, 16])
def test_bits_plane_multi_hit(V, oracle_lib, monkeypatch, k):
    """vsr_trace_multi reads the plane too: same bytes as the A8 path (which test_gpu_multi.py
    checks against walker C)."""
    o = oracle_lib
    sc = soup_with([(64, 96), (32, 160), (128, 128)], seed=95)
    rays = W.random_rays(8011, seed=96).data
    s = V.Scene.from_workload(sc).build()
    r = torch.from_numpy(np.ascontiguousarray(rays, np.float32)).cuda()
    out = {}
    for bits in (True, False):
        monkeypatch.setenv("VSR_ALPHA_BITS", "1" if bits else "0")
        h, nh, _ = s.trace_multi(r, k, V.ALPHA_TEXTURE, alpha_threshold=0.5)
        torch.cuda.synchronize()
        out[bits] = (h.cpu().numpy().tobytes(), nh.cpu().numpy().tobytes())
    assert out[True] == out[False]


def test_bits_plane_in_lists_and_instances(V, monkeypatch):
    """Lists and instances read every element's plane (all elements 32-aligned), or all fall back
    to A8 when one is not; bytes equal to the A8 path in both cases, any / closest / multi-hit."""
    aligned = [soup_with([(64, 96), (32, 160)], seed=97), soup_with([(128, 64)], seed=98)]
    mixed = aligned[:1] + [soup_with([(24, 40)], seed=99)]
    models, ibvh, imat = W.instanced_forest(n_instances=400, n_models=2, cards=16)
    rays = W.random_rays(6007, seed=100).data
    r = torch.from_numpy(np.ascontiguousarray(rays, np.float32)).cuda()
    _, frame = W.config("C2", 240, 136)
    fr = torch.from_numpy(frame.data).cuda()
    for elems in (aligned, mixed):
        scenes = [V.Scene.from_workload(e).build() for e in elems]
        grp = V.Group(scenes)
        out = {}
        for bits in (True, False):
            monkeypatch.setenv("VSR_ALPHA_BITS", "1" if bits else "0")
            res = []
            for q in (V.ANY, V.CLOSEST):
                h, w, _ = grp.trace(r, q, V.ALPHA_TEXTURE, alpha_threshold=0.4)
                res += [h.cpu().numpy().tobytes(), w.cpu().numpy().tobytes()]
            mh, mn, mw, _ = grp.trace_multi(r, 4, V.ALPHA_TEXTURE, alpha_threshold=0.4)
            res += [mh.cpu().numpy().tobytes(), mn.cpu().numpy().tobytes()]
            out[bits] = res
        assert out[True] == out[False]
    mscenes = [V.Scene.from_workload(m).build() for m in models]
    inst = V.Instances(mscenes, ibvh, imat)
    out = {}
    for bits in (True, False):
        monkeypatch.setenv("VSR_ALPHA_BITS", "1" if bits else "0")
        res = []
        for q in (V.ANY, V.CLOSEST):
            h, w, _ = inst.trace(fr, q, V.ALPHA_TEXTURE, alpha_threshold=0.3)
            res += [h.cpu().numpy().tobytes(), w.cpu().numpy().tobytes()]
        out[bits] = res
    assert out[True] == out[False]
