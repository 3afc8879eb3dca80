"""Randomised parity sweep over scales and offsets (-m gpu): scenes scaled by 1e-3..1e4 and
moved up to 1e5 away from the origin, rays with tiny, huge and axis-parallel directions and
assorted [tmin, tmax].  GPU == walker C bit for bit (hits, counts) on the product's BVH, and
GPU == brute force (hit/miss exact, prims up to exact ties) — the second half is the BVH's
conservativeness: the padded boxes and the widened slab exit must never cull a triangle that
Möller–Trumbore accepts."""
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


def fuzz_case(seed):
    rng = np.random.default_rng(1000 + seed)
    scale = 10.0 ** rng.uniform(-3, 4)
    offset = rng.uniform(-1, 1, 3) * 10.0 ** rng.uniform(2, 6) if seed % 2 else np.zeros(3)
    n = int(rng.integers(200, 1500))
    sc = W.random_soup(n, seed=2000 + seed, extent=10.0, size=float(rng.uniform(0.05, 3.0)))
    sc.vertices = (sc.vertices.astype(np.float64).reshape(-1, 3) * scale + offset).reshape(-1, 9)
    sc.vertices = sc.vertices.astype(np.float32)
    m = 4096 + int(rng.integers(0, 128))        # ragged tail
    rays = W.random_rays(m, seed=3000 + seed, extent=14.0, target=8.0).data.astype(np.float64)
    rays[:, 0:3] = rays[:, 0:3] * scale + offset
    d = rays[:, 4:7]
    k = rng.random(m)
    d[k < 0.1] *= 1e-20                         # tiny directions (t scales up)
    d[(k >= 0.1) & (k < 0.2)] *= 1e15           # huge directions
    ax = (k >= 0.2) & (k < 0.35)                # axis-parallel: zero two components
    keep = rng.integers(0, 3, m)
    for a in range(3):
        d[ax & (keep != a), a] = 0.0
    rays[:, 4:7] = d
    tmax = np.where(rng.random(m) < 0.2, rng.uniform(0.0, 30.0, m) * scale / np.maximum(
        np.linalg.norm(d, axis=1), 1e-30), np.inf)
    rays[:, 7] = tmax
    rays[:, 3] = np.where(rng.random(m) < 0.1, 0.0, 1e-4)
    return sc, rays.astype(np.float32)


@pytest.mark.parametrize("seed", range(16))
def test_fuzz_scale_offset(V, oracle_lib, seed):
    o = oracle_lib
    sc, rays = fuzz_case(seed)
    assert np.all(np.isfinite(rays[:, 0:7]))
    s = V.Scene.from_workload(sc).build(max_leaf_size=1 + seed % 4)
    b = bvh_check.to_oracle(s.export())
    r = torch.from_numpy(rays).cuda()
    for q, oq in ((V.CLOSEST, o.CLOSEST), (V.ANY, o.ANY)):
        for k, ok in ((V.COUNT, o.DEFAULT), (V.COUNT_ALPHA_TEXTURE, o.ALPHA_TEX),
                      (V.ALPHA_PROCEDURAL, o.ALPHA_PROC)):
            h, c = s.trace(r, q, k)
            torch.cuda.synchronize()
            h = V.hits_to_numpy(h)
            wh, wc = o.walk(b, rays, oq, ok)
            assert np.array_equal(h.view(np.uint32), wh.view(np.uint32)), (seed, q, k)
            if c is not None:
                c = V.counts_to_numpy(c)
                assert np.array_equal(c["boxes"], wc["boxes"]) and np.array_equal(c["tris"], wc["tris"])
            ref, nt = o.trace(sc, rays, oq, ok, ties=True)
            compare(o, sc, rays, oq, ok, h, ref, nt)
