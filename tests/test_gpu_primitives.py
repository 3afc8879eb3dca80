"""Query on a plain list of primitives (vsr_trace_primitives): the brute-force
definition itself, so the GPU must equal oracle S on EVERY ray, exact ties included (lowest
index for closest, lowest accepted index for any-hit), for every intersector kind; counts are
the triangle tests made (no boxes)."""
import numpy as np
import pytest

import workloads as W

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


KINDS = (("NONE", "NONE"), ("DEFAULT", "DEFAULT"), ("ALPHA_TEXTURE", "ALPHA_TEX"),
         ("ALPHA_PROCEDURAL", "ALPHA_PROC"), ("ALPHA_TEXTURE_BILINEAR", "ALPHA_TEX_BILINEAR"),
         ("ALPHA_PROCEDURAL_UV", "ALPHA_PROC_UV"))


def with_duplicates(sc, k):
    """Append copies of the first k triangles (exact ties in t) and one degenerate triangle."""
    v = np.concatenate([sc.vertices, sc.vertices[:k]])
    d = v[:1].copy()
    d[0, 3:6] = d[0, 0:3]
    v = np.concatenate([v, d])
    g = np.concatenate([sc.geom_ids, sc.geom_ids[:k], sc.geom_ids[:1]])
    t = np.concatenate([sc.texcoords, sc.texcoords[:k], sc.texcoords[:1]])
    return W.Scene("dup", v.astype(np.float32), g, t, sc.geom_texture, sc.textures)


@pytest.mark.parametrize("n_tris", [1, 130, 700])
def test_primitives_equal_bruteforce_exactly(V, oracle_lib, n_tris):
    o = oracle_lib
    sc = with_duplicates(W.random_soup(n_tris, seed=100 + n_tris, size=2.5), min(n_tris, 60))
    rays = W.random_rays(1537, seed=101).data          # ragged: 12 blocks + 1 ray
    s = V.Scene.from_workload(sc).build()
    r = torch.from_numpy(rays).cuda()
    valid = sc.num_tris - 1                              # the degenerate one is excluded
    for vq, oq in ((V.CLOSEST, o.CLOSEST), (V.ANY, o.ANY)):
        for vk, ok in KINDS:
            h, _ = s.trace_primitives(r, vq, getattr(V, vk), alpha_threshold=0.3, checker_freq=5)
            torch.cuda.synchronize()
            h = V.hits_to_numpy(h)
            ref = o.trace(sc, rays, oq, getattr(o, ok), alpha_threshold=0.3, checker_freq=5)
            assert np.array_equal(h.view(np.uint32), ref.view(np.uint32)), (vq, vk)
        h, c = s.trace_primitives(r, vq, V.COUNT_ALPHA_TEXTURE)
        torch.cuda.synchronize()
        c = V.counts_to_numpy(c)
        assert np.all(c["boxes"] == 0)
        if vq == V.CLOSEST:
            assert np.all(c["tris"] == valid)
        else:
            assert np.all(c["tris"] <= valid)


def test_primitives_match_the_bvh_on_c1(V, oracle_lib):
    sc, rays = W.config("C1")
    s = V.Scene.from_workload(sc).build()
    r = torch.from_numpy(rays.data).cuda()
    a, _ = s.trace_primitives(r, V.CLOSEST, V.ALPHA_TEXTURE)
    b, _ = s.trace(r, V.CLOSEST, V.ALPHA_TEXTURE)
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
