"""GPU parity: the CUDA path through the C ABI vs the CPU oracle (-m gpu).

* oracle S (brute force) decides hits: element by element on small scenes
  spanning many 128-ray blocks with a ragged tail, and on seeded samples of
  the full-size C2 frame traced in the bench's launch configuration;
* walker C decides counts: bit-exact on an oracle-built BVH imported into
  the product, and on the product's own exported BVH (full frame);
* invariants that hold at any size are checked on whole frames.
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


def oracle_kind(V, o, isect):
    base = isect % 100 if isect >= 100 else isect
    return {V.NONE: o.NONE, V.DEFAULT: o.DEFAULT, V.ALPHA_TEXTURE: o.ALPHA_TEX,
            V.ALPHA_PROCEDURAL: o.ALPHA_PROC, V.COUNT: o.DEFAULT,
            V.COUNT_ALPHA_TEXTURE: o.ALPHA_TEX}[base]


ALL_KINDS = ["NONE", "DEFAULT", "ALPHA_TEXTURE", "ALPHA_PROCEDURAL", "COUNT", "COUNT_ALPHA_TEXTURE",
             "RUNTIME_SWITCH_DEFAULT", "RUNTIME_SWITCH_ALPHA_TEXTURE",
             "RUNTIME_SWITCH_ALPHA_PROCEDURAL", "RUNTIME_FNPTR_DEFAULT",
             "RUNTIME_FNPTR_ALPHA_TEXTURE", "RUNTIME_FNPTR_ALPHA_PROCEDURAL"]


def gpu_trace(V, scene, rays_np, query, isect, **kw):
    r = torch.from_numpy(np.ascontiguousarray(rays_np, np.float32)).cuda()
    hits, counts = scene.trace(r, query=query, isect=isect, **kw)
    torch.cuda.synchronize()
    h = V.hits_to_numpy(hits)
    c = V.counts_to_numpy(counts) if counts is not None else None
    return h, c


def check_against_oracle(V, o, wl_scene, scene, rays_np, query, isect, **kw):
    h, c = gpu_trace(V, scene, rays_np, query, isect, **kw)
    ok = oracle_kind(V, o, isect)
    okw = {}
    if "alpha_threshold" in kw:
        okw["alpha_threshold"] = kw["alpha_threshold"]
    if "checker_freq" in kw:
        okw["checker_freq"] = kw["checker_freq"]
    ref, nt = o.trace(wl_scene, rays_np, query=query, isect=ok, ties=True, **okw)
    summary = compare(o, wl_scene, rays_np, query, ok, h, ref, nt, **okw)
    return h, c, summary


@pytest.mark.parametrize("query", ["CLOSEST", "ANY"])
@pytest.mark.parametrize("kind", ALL_KINDS)
def test_c1_all_kinds(V, oracle_lib, query, kind):
    sc, rays = W.config("C1")
    s = V.Scene.from_workload(sc).build(max_leaf_size=1)
    q, k = getattr(V, query), getattr(V, kind)
    h, c, summ = check_against_oracle(V, oracle_lib, sc, s, rays.data, q, k)
    assert summ["hits"] > 0
    if c is not None:   # counts bit-exact vs walker C on the same (exported) BVH
        b = bvh_check.to_oracle(s.export())
        wh, wc = oracle_lib.walk(b, rays.data, query=q, isect=oracle_kind(V, oracle_lib, k))
        assert np.array_equal(c["boxes"], wc["boxes"]) and np.array_equal(c["tris"], wc["tris"])
        assert np.array_equal(c["alpha"], wc["alpha"])
        assert np.array_equal(h, wh)


@pytest.mark.parametrize("max_leaf", [1, 4, 16])
@pytest.mark.parametrize("n_rays", [1, 31, 129, 5000])
def test_soup_parity_ragged(V, oracle_lib, max_leaf, n_rays):
    sc = W.random_soup(1500, seed=100 + max_leaf)
    rays = W.random_rays(n_rays, seed=200 + n_rays)
    s = V.Scene.from_workload(sc).build(max_leaf_size=max_leaf)
    for q in (V.CLOSEST, V.ANY):
        for k in (V.NONE, V.DEFAULT, V.ALPHA_TEXTURE, V.ALPHA_PROCEDURAL):
            check_against_oracle(V, oracle_lib, sc, s, rays.data, q, k)


def test_params_threshold_and_checker(V, oracle_lib):
    sc = W.random_soup(800, seed=7)
    rays = W.random_rays(3000, seed=8)
    s = V.Scene.from_workload(sc).build()
    for thr in (0.0, 0.01, 3 / 255, 0.5, 1.0, 1.5):
        check_against_oracle(V, oracle_lib, sc, s, rays.data, V.CLOSEST, V.ALPHA_TEXTURE,
                             alpha_threshold=thr)
    for m in (1, 2, 3, 8, 13):
        check_against_oracle(V, oracle_lib, sc, s, rays.data, V.CLOSEST, V.ALPHA_PROCEDURAL,
                             checker_freq=m)


def test_edge_rays(V, oracle_lib):
    """Axis-parallel directions (zero components), origins inside boxes, empty
    [tmin, tmax] intervals, tmax cutting the scene, rays that miss."""
    sc = W.stacked_quads(5)
    rng = np.random.default_rng(9)
    rays = []
    for _ in range(600):
        o = rng.uniform(-0.5, 1.5, 3)
        o[2] = rng.choice([-1.0, 2.5, 7.0])
        d = np.zeros(3)
        d[2] = rng.choice([-1.0, 1.0, 0.0])
        if rng.random() < 0.3:
            d[0] = rng.normal() * 0.2
        if not d.any():
            d[1] = 1.0
        tmin = rng.choice([1e-4, 0.0, 1.5])
        tmax = rng.choice([np.inf, 2.0, 1.0, tmin])
        rays.append([*o, tmin, *d, tmax])
    rays = np.array(rays, np.float32)
    s = V.Scene.from_workload(sc).build(max_leaf_size=2)
    for q in (V.CLOSEST, V.ANY):
        for k in (V.DEFAULT, V.ALPHA_PROCEDURAL):
            check_against_oracle(V, oracle_lib, sc, s, rays, q, k)


@pytest.mark.parametrize("refill", ["32", "8"])
def test_persistent_schedule(V, oracle_lib, monkeypatch, refill):
    """The persistent dynamic-fetch kernel gives the same bytes as the direct one;
    its self-resetting work counters survive > 256 launches (slot reuse)."""
    sc = W.random_soup(1500, seed=5)
    rays = W.random_rays(5003, seed=6)
    s = V.Scene.from_workload(sc).build()
    ref = {}
    for q in (V.CLOSEST, V.ANY):
        for k in (V.DEFAULT, V.ALPHA_TEXTURE, V.COUNT_ALPHA_TEXTURE):
            ref[(q, k)] = gpu_trace(V, s, rays.data, q, k)
    monkeypatch.setenv("VSR_SCHED", "persistent")
    monkeypatch.setenv("VSR_REFILL", refill)
    for q in (V.CLOSEST, V.ANY):
        for k in (V.DEFAULT, V.ALPHA_TEXTURE, V.COUNT_ALPHA_TEXTURE):
            h, c = check_against_oracle(V, oracle_lib, sc, s, rays.data, q, k)[:2]
            assert h.tobytes() == ref[(q, k)][0].tobytes()
            if c is not None:
                assert c.tobytes() == ref[(q, k)][1].tobytes()
    r = torch.from_numpy(rays.data).cuda()
    hits = torch.empty((rays.n, 4), device="cuda")
    for _ in range(300):
        s.trace(r, V.CLOSEST, V.ALPHA_TEXTURE, hits=hits)
    torch.cuda.synchronize()
    assert V.hits_to_numpy(hits).tobytes() == ref[(V.CLOSEST, V.ALPHA_TEXTURE)][0].tobytes()


@pytest.mark.parametrize("knobs", [{"VSR_ORDER": "0"}, {"VSR_PDL": "0"},
                                   {"VSR_ORDER": "0", "VSR_ALPHA_BITS": "0"}, {"VSR_OCC": "1"},
                                   {"VSR_SCHED": "warp"}, {"VSR_SCHED": "warp", "VSR_OCC": "1"},
                                   {"VSR_SCHED": "warp", "VSR_ORDER": "0"},
                                   {"VSR_SCHED": "region"}, {"VSR_SCHED": "region", "VSR_OCC": "1"},
                                   {"VSR_ORDER_PROXY": "grid"}, {"VSR_ORDER_PROXY": "len"},
                                   {"VSR_ORDER_PROXY": "mix"}])
def test_scheduling_knobs_change_no_result(V, c2, monkeypatch, knobs):
    """README's runtime knobs: tile order instead of longest-first, plain launches instead of
    the PDL chain, A8 instead of the 1-bit plane, the closest-hit occupancy variant — the same
    bytes as the defaults (C2 frame, large enough for the order pass to run)."""
    sc, rays, s = c2
    ref = {}
    for q in (V.CLOSEST, V.ANY):
        for k in (V.ALPHA_TEXTURE, V.COUNT_ALPHA_TEXTURE):
            ref[(q, k)] = gpu_trace(V, s, rays.data, q, k)
    for name, val in knobs.items():
        monkeypatch.setenv(name, val)
    for q in (V.CLOSEST, V.ANY):
        for k in (V.ALPHA_TEXTURE, V.COUNT_ALPHA_TEXTURE):
            h, c = gpu_trace(V, s, rays.data, q, k)
            assert h.tobytes() == ref[(q, k)][0].tobytes(), (knobs, q, k)
            if c is not None:
                assert c.tobytes() == ref[(q, k)][1].tobytes()


def test_imported_oracle_bvh_counts(V, oracle_lib):
    """Counts bit-exact on a tree the product did NOT build (oracle median BVH)."""
    o = oracle_lib
    sc = W.random_soup(3000, seed=301)
    rays = W.random_rays(20000, seed=302)
    b = o.build_bvh(sc, max_leaf=4)
    arrs = {"root_ref": b.root_ref, "root_lo": b.root_lo, "root_hi": b.root_hi, "nodes": b.nodes,
            "tris": b.tris, "sides": b.sides, "texdescs": b.texdescs, "texels": b.texels}
    s = V.Scene.import_arrays(arrs)
    for q in (V.CLOSEST, V.ANY):
        for k, ok in ((V.COUNT, o.DEFAULT), (V.COUNT_ALPHA_TEXTURE, o.ALPHA_TEX)):
            h, c = gpu_trace(V, s, rays.data, q, k)
            wh, wc = o.walk(b, rays.data, query=q, isect=ok)
            assert np.array_equal(h, wh)
            assert np.array_equal(c["boxes"], wc["boxes"])
            assert np.array_equal(c["tris"], wc["tris"])
            assert np.array_equal(c["alpha"], wc["alpha"])


def test_errors(V):
    sc = W.quad_pair_scene()
    s = V.Scene.from_workload(sc)
    r = torch.zeros((4, 8), device="cuda")
    with pytest.raises(V.VsrError) as e:
        s.trace(r)
    assert e.value.status == V.ERR_NOT_BUILT
    s.build()
    hits = torch.empty((4, 4), device="cuda")
    with pytest.raises(V.VsrError) as e:   # COUNT without a counts buffer
        s.trace_raw(r.data_ptr(), 4, V.CLOSEST, V.COUNT, hits.data_ptr(), None)
    assert e.value.status == V.ERR_INVALID_ARG
    buf = torch.zeros(4 * 8 + 4, device="cuda")
    with pytest.raises(V.VsrError) as e:
        s.trace_raw(buf.data_ptr() + 4, 4, V.CLOSEST, V.DEFAULT,
                    torch.empty((4, 4), device="cuda").data_ptr())
    assert e.value.status == V.ERR_INVALID_ARG
    with pytest.raises(V.VsrError) as e:
        s.trace_raw(r.data_ptr(), 4, 7, V.DEFAULT, torch.empty((4, 4), device="cuda").data_ptr())
    assert e.value.status == V.ERR_INVALID_ARG
    n0 = V.launch_count()
    s.trace_raw(r.data_ptr(), 0, V.CLOSEST, V.DEFAULT, 0)   # n = 0 is a no-op
    assert V.launch_count() == n0


# ---------------------------------------------------------------------------
# full-size C2 (BASELINE.json configs[1]) in the bench's launch configuration
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def c2(V):
    sc, rays = W.config("C2")
    s = V.Scene.from_workload(sc).build()
    return sc, rays, s


def test_c2_sampled_parity(V, oracle_lib, c2):
    """262,144 seeded rays of the full C2 frame against oracle S for both
    queries x {default, alpha texture, procedural}; every returned any-hit is validated."""
    sc, rays, s = c2
    osc = oracle_lib.OracleScene(sc)
    idx = np.sort(np.random.default_rng(2024).choice(rays.n, 262144, replace=False))
    sub = np.ascontiguousarray(rays.data[idx])
    for q in (V.CLOSEST, V.ANY):
        for k in (V.DEFAULT, V.ALPHA_TEXTURE, V.ALPHA_PROCEDURAL):
            h, _ = gpu_trace(V, s, rays.data, q, k)     # the whole frame, one launch
            ok = oracle_kind(V, oracle_lib, k)
            if q == V.CLOSEST:
                ref, nt = oracle_lib.trace(osc, sub, query=q, isect=ok, ties=True)
            else:   # any-hit needs no tie count: every returned hit is validated instead
                ref, nt = oracle_lib.trace(osc, sub, query=q, isect=ok), None
            compare(oracle_lib, osc, sub, q, ok, h[idx], ref, nt)


def test_c2_full_frame_invariants(V, oracle_lib, c2):
    sc, rays, s = c2
    hn, _ = gpu_trace(V, s, rays.data, V.CLOSEST, V.NONE)
    hd, _ = gpu_trace(V, s, rays.data, V.CLOSEST, V.DEFAULT)
    assert hn.tobytes() == hd.tobytes()            # zero-cost: byte-identical
    ha, _ = gpu_trace(V, s, rays.data, V.CLOSEST, V.ALPHA_TEXTURE)
    hany, _ = gpu_trace(V, s, rays.data, V.ANY, V.ALPHA_TEXTURE)
    hc, cc = gpu_trace(V, s, rays.data, V.CLOSEST, V.COUNT)
    assert hc.tobytes() == hd.tobytes()            # counting is observationally pure
    dh, ah = hd["prim"] != 0xFFFFFFFF, ha["prim"] != 0xFFFFFFFF
    assert np.all(dh[ah]) and ah.sum() < dh.sum()  # masks only clear hits
    assert np.array_equal(ah, hany["prim"] != 0xFFFFFFFF)
    assert 0.05 < ah.mean() < 0.95
    # counts over the full frame vs walker C on the exported BVH (bit-exact)
    b = bvh_check.to_oracle(s.export())
    wh, wc = oracle_lib.walk(b, rays.data, isect=oracle_lib.DEFAULT)
    assert np.array_equal(cc["boxes"], wc["boxes"]) and np.array_equal(cc["tris"], wc["tris"])
    assert hd.tobytes() == wh.tobytes()
    _, ca = gpu_trace(V, s, rays.data, V.CLOSEST, V.COUNT_ALPHA_TEXTURE)
    wha, wca = oracle_lib.walk(b, rays.data, isect=oracle_lib.ALPHA_TEX)
    assert ha.tobytes() == wha.tobytes()
    for f in ("boxes", "tris", "alpha"):
        assert np.array_equal(ca[f], wca[f])


def test_c2_trace_host_equals_device(V, c2):
    sc, rays, s = c2
    for k in (V.ALPHA_TEXTURE, V.COUNT):
        hd, cd = gpu_trace(V, s, rays.data, V.CLOSEST, k)
        pinned = torch.from_numpy(rays.data).pin_memory()
        hh, ch = s.trace_host(pinned, V.CLOSEST, k)
        assert hh.tobytes() == hd.tobytes()
        if cd is not None:
            assert ch.tobytes() == cd.tobytes()


@pytest.mark.parametrize("chunk,pin", [("4096", True), ("65536", True), ("300000", True),
                                       ("4096", False)])
def test_trace_host_ring_reuse(V, c2, monkeypatch, chunk, pin):
    """The host pipeline's ring of 8 chunk slots: more chunks than slots (slot reuse behind
    the D2H event), a ragged last chunk, counts and hits both staged, pinned or pageable rays
    (hits: pageable numpy); equal to the device path."""
    sc, rays, s = c2
    sub = np.ascontiguousarray(rays.data[: 8 * 4096 * 3 + 777])   # 99,081 rays
    monkeypatch.setenv("VSR_HOST_CHUNK", chunk)
    pinned = torch.from_numpy(sub).pin_memory() if pin else sub
    for q, k in ((V.ANY, V.ALPHA_TEXTURE), (V.CLOSEST, V.COUNT_ALPHA_TEXTURE), (V.ANY, V.COUNT)):
        hd, cd = gpu_trace(V, s, sub, q, k)
        hh, ch = s.trace_host(pinned, q, k)
        assert hh.tobytes() == hd.tobytes(), (chunk, q, k)
        if cd is not None:
            assert ch.tobytes() == cd.tobytes(), (chunk, q, k)


def test_tile_sharding_is_partition_invariant(V, c2):
    """Fake-P emulation of the multi-GPU deal (tile k -> rank k mod P): tracing
    each rank's shard separately and scattering back is byte-identical to P=1."""
    sc, rays, s = c2
    full, _ = gpu_trace(V, s, rays.data, V.CLOSEST, V.ALPHA_TEXTURE)
    from paper_1912_12786_b200 import shard
    for P in (2, 4, 8):
        out = np.empty_like(full)
        for rank in range(P):
            idx = shard.rank_ray_indices(rays.n, 64, rank, P)
            h, _ = gpu_trace(V, s, rays.data[idx], V.CLOSEST, V.ALPHA_TEXTURE)
            out[idx] = h
        assert out.tobytes() == full.tobytes()


@pytest.mark.parametrize("sched", ["warp", "region"])
@pytest.mark.parametrize("n", [1, 31, 33, 129, 5000, 40000, 40017])
def test_warp_schedule_ragged(V, oracle_lib, monkeypatch, n, sched):
    """VSR_SCHED=warp (32-ray chunks claimed per warp, next chunk prefetched) and
    VSR_SCHED=region (chunks claimed from the SM's own block range, stealing when it is
    empty; engaged from 2 x 148 blocks): ragged ray counts (a partial chunk, fewer chunks
    than warps, ragged regions) give the direct schedule's bytes."""
    sc = W.random_soup(2000, seed=900 + n)
    rays = W.random_rays(n, seed=901 + n).data
    s = V.Scene.from_workload(sc).build()
    ref = {q: gpu_trace(V, s, rays, q, V.COUNT_ALPHA_TEXTURE) for q in (V.CLOSEST, V.ANY)}
    monkeypatch.setenv("VSR_SCHED", sched)
    for q in (V.CLOSEST, V.ANY):
        # poisoned outputs: a ray the schedule never traces cannot inherit a stale row
        hits = torch.full((n, 4), float("nan"), device="cuda")
        counts = torch.full((n, 4), -1, dtype=torch.int32, device="cuda")
        h, c = gpu_trace(V, s, rays, q, V.COUNT_ALPHA_TEXTURE, hits=hits, counts=counts)
        assert h.tobytes() == ref[q][0].tobytes() and c.tobytes() == ref[q][1].tobytes()
