"""GPU parity on the large configs (BASELINE.json configs[3], configs[4]):

* C4 — 1M-triangle terrain + billboards, 1080p: the counting intersector over
  the full frame bit-exact against walker C on the exported BVH; hits against
  oracle S (brute force over all 1.04 M triangles) on a 16,384-ray seeded sample.
* C5 — 10.2M triangles, 3840×2160×4 spp (33.2 M rays, one launch): hits against
  oracle S on a 16,384-ray seeded sample; counts against walker C on a 1 M-ray sample.
"""
import numpy as np
import pytest

import workloads as W
from tests import bvh_check
from tests.parity import compare

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


@pytest.fixture(scope="module")
def textures():
    return W.tree_textures(16, 1024, 2)


def _trace(V, s, d_rays, q, k):
    hits, counts = s.trace(d_rays, query=q, isect=k)
    torch.cuda.synchronize()
    h = V.hits_to_numpy(hits)
    c = V.counts_to_numpy(counts) if counts is not None else None
    del hits, counts
    return h, c


def test_c4_counts_full_frame_and_sampled_hits(V, oracle_lib, textures):
    o = oracle_lib
    sc, rays = W.scene("C4", textures), W.rays_for("C4")
    s = V.Scene.from_workload(sc).build()
    d = torch.from_numpy(rays.data).cuda()
    h, c = _trace(V, s, d, V.CLOSEST, V.COUNT)
    hd, _ = _trace(V, s, d, V.CLOSEST, V.DEFAULT)
    assert h.tobytes() == hd.tobytes()
    b = bvh_check.to_oracle(s.export())
    wh, wc = o.walk(b, rays.data, isect=o.DEFAULT)
    assert np.array_equal(c["boxes"], wc["boxes"]) and np.array_equal(c["tris"], wc["tris"])
    assert h.tobytes() == wh.tobytes()
    assert (h["prim"] != 0xFFFFFFFF).mean() > 0.3          # the terrain fills the frame
    idx = np.sort(np.random.default_rng(44).choice(rays.n, 16384, replace=False))
    sub = np.ascontiguousarray(rays.data[idx])
    osc = o.OracleScene(sc)
    for k, ok in ((V.DEFAULT, o.DEFAULT), (V.ALPHA_TEXTURE, o.ALPHA_TEX)):
        for q, oq in ((V.CLOSEST, o.CLOSEST), (V.ANY, o.ANY)):
            g, _ = _trace(V, s, d, q, k)
            ref, nt = (o.trace(osc, sub, query=oq, isect=ok, ties=True) if oq == o.CLOSEST
                       else (o.trace(osc, sub, query=oq, isect=ok), None))
            compare(o, osc, sub, oq, ok, g[idx], ref, nt)


def test_c5_full_launch_sampled_parity(V, oracle_lib, textures):
    o = oracle_lib
    sc, rays = W.scene("C5", textures), W.rays_for("C5")
    assert rays.n == 3840 * 2160 * 4
    s = V.Scene.from_workload(sc).build()
    d = torch.from_numpy(rays.data).cuda()
    idx = np.sort(np.random.default_rng(55).choice(rays.n, 16384, replace=False))
    sub = np.ascontiguousarray(rays.data[idx])
    osc = o.OracleScene(sc)
    for q, oq in ((V.CLOSEST, o.CLOSEST), (V.ANY, o.ANY)):
        g, _ = _trace(V, s, d, q, V.ALPHA_TEXTURE)
        ref, nt = (o.trace(osc, sub, query=oq, isect=o.ALPHA_TEX, ties=True) if oq == o.CLOSEST
                   else (o.trace(osc, sub, query=oq, isect=o.ALPHA_TEX), None))
        compare(o, osc, sub, oq, o.ALPHA_TEX, g[idx], ref, nt)
    sub = np.sort(np.random.default_rng(56).choice(rays.n, 1 << 20, replace=False))
    h, c = _trace(V, s, d, V.CLOSEST, V.COUNT_ALPHA_TEXTURE)
    b = bvh_check.to_oracle(s.export())
    wh, wc = o.walk(b, rays.data[sub], isect=o.ALPHA_TEX)
    assert h[sub].tobytes() == wh.tobytes()
    for f in ("boxes", "tris", "alpha"):
        assert np.array_equal(c[f][sub], wc[f])
