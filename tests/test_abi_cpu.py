"""CPU-only tests of the product library: it loads, exports every symbol that
include/vsr.h declares, validates arguments as documented, and its host BVH
builder produces valid trees that prune exactly (checked with the oracle's
contract walker against brute force).  No kernel is launched here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import workloads as W
from tests import bvh_check

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def vsr():
    from paper_1912_12786_b200 import _build
    _build.build()
    from paper_1912_12786_b200 import vsr as V
    return V


def test_header_symbols_exported(vsr):
    hdr = open(os.path.join(ROOT, "include", "vsr.h")).read()
    declared = sorted(set(re.findall(r"^\s*(?:vsr_status|const char\*|uint64_t|uint32_t)\s+(vsr_\w+)\s*\(",
                                     hdr, re.M)))
    assert len(declared) >= 11
    assert set(declared) == set(vsr.EXPORTED_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", vsr.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (vsr_\w+)", out))
    for name in declared:
        assert name in exported, name
        assert hasattr(vsr.lib(), name)
    assert vsr.lib().vsr_abi_version() == 2


def test_library_is_sm100a(vsr):
    out = subprocess.run(["cuobjdump", "--list-elf", vsr.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _err(vsr, fn):
    with pytest.raises(vsr.VsrError) as ei:
        fn()
    return ei.value.status


def test_create_validation(vsr):
    sc = W.quad_pair_scene()
    v = sc.vertices.copy()
    v[1, 4] = np.nan
    assert _err(vsr, lambda: vsr.Scene(v, device=-1)) == vsr.ERR_NONFINITE
    tc = sc.texcoords.copy()
    tc[0, 0] = np.inf
    assert _err(vsr, lambda: vsr.Scene(sc.vertices, texcoords=tc, device=-1)) == vsr.ERR_NONFINITE
    tc = sc.texcoords.copy()
    tc[0, 0] = 2000.0
    assert _err(vsr, lambda: vsr.Scene(sc.vertices, texcoords=tc, device=-1)) == vsr.ERR_INVALID_ARG
    # geom -> texture out of range
    assert _err(vsr, lambda: vsr.Scene(sc.vertices, sc.geom_ids, sc.texcoords,
                                       np.array([0, 5], np.uint32), sc.textures,
                                       device=-1)) == vsr.ERR_INVALID_ARG
    # geom id beyond num_geoms
    assert _err(vsr, lambda: vsr.Scene(sc.vertices, np.array([0, 0, 1, 7], np.uint32),
                                       sc.texcoords, sc.geom_texture, sc.textures,
                                       device=-1)) == vsr.ERR_INVALID_ARG
    # NULL desc / NULL out
    h = C.c_void_p()
    assert vsr.lib().vsr_scene_create(None, C.byref(h)) == vsr.ERR_INVALID_ARG
    assert vsr.lib().vsr_last_error().decode() != ""
    assert vsr.lib().vsr_destroy(None) == vsr.OK


def test_build_validation(vsr):
    empty = vsr.Scene(np.zeros((0, 9), np.float32), device=-1)
    assert _err(vsr, lambda: empty.build()) == vsr.ERR_EMPTY_SCENE
    degen = np.tile(np.array([[0, 0, 0, 1, 1, 1, 2, 2, 2]], np.float32), (5, 1))
    assert _err(vsr, lambda: vsr.Scene(degen, device=-1).build()) == vsr.ERR_EMPTY_SCENE
    sc = vsr.Scene.from_workload(W.quad_pair_scene(), device=-1)
    assert _err(vsr, lambda: sc.build(max_leaf_size=0)) == vsr.ERR_INVALID_ARG
    assert _err(vsr, lambda: sc.build(max_leaf_size=33)) == vsr.ERR_INVALID_ARG
    assert _err(vsr, lambda: sc.build(sah_bins=1)) == vsr.ERR_INVALID_ARG
    # trace before build / on a host-only scene
    h = np.zeros((4, 8), np.float32)
    assert _err(vsr, lambda: sc.trace_host(h)) == vsr.ERR_UNSUPPORTED
    sc.build()
    assert sc.stats()["built"] == 1


def test_degenerate_excluded(vsr):
    sc = W.random_soup(50, seed=3)
    v = sc.vertices.copy()
    v[7, 3:6] = v[7, 0:3]          # zero-length edge
    v[9, 6:9] = 2 * v[9, 3:6] - v[9, 0:3]   # collinear: v2 = v0 + 2 e1 (exact in most cases)
    s = vsr.Scene(v, sc.geom_ids, sc.texcoords, sc.geom_texture, sc.textures, device=-1).build()
    st = s.stats()
    assert st["num_degenerate"] >= 1 and st["num_tris"] == 50 - st["num_degenerate"]
    e = s.export()
    assert 7 not in set(e["tris"][:, 3].tolist())


@pytest.mark.parametrize("max_leaf", [1, 4, 16])
def test_product_bvh_valid(vsr, max_leaf):
    sc = W.random_soup(3000, seed=71)
    s = vsr.Scene.from_workload(sc, device=-1).build(max_leaf_size=max_leaf)
    e = s.export()
    d = bvh_check.validate(e, sc.vertices, max_leaf)
    assert d == s.stats()["max_depth"]
    assert e["nodes"].shape[0] == s.stats()["num_nodes"]


def test_single_triangle_and_coincident(vsr):
    one = W.stacked_quads(1)
    one.vertices = one.vertices[:1]
    one.geom_ids = one.geom_ids[:1]
    one.texcoords = one.texcoords[:1]
    s = vsr.Scene.from_workload(one, device=-1).build()
    e = s.export()
    assert e["nodes"].shape[0] == 0 and e["root_ref"] & 0x80000000
    lo = one.vertices[0].reshape(3, 3).min(0)
    hi = one.vertices[0].reshape(3, 3).max(0)
    assert np.all(e["root_lo"] <= lo) and np.all(e["root_hi"] >= hi)
    assert np.all(e["root_lo"] >= lo - 1e-5) and np.all(e["root_hi"] <= hi + 1e-5)
    n = 1000
    same = np.tile(np.array([[0, 0, 0, 1, 0, 0, 0, 1, 0]], np.float32), (n, 1))
    s = vsr.Scene(same, device=-1).build()
    d = bvh_check.validate(s.export(), same, 4)
    assert d <= int(np.ceil(np.log2(n))) + 1


def _walker_vs_bruteforce(vsr, oracle_lib, sc, rays, isects, max_leaf=4):
    s = vsr.Scene.from_workload(sc, device=-1).build(max_leaf_size=max_leaf)
    b = bvh_check.to_oracle(s.export())
    for isect in isects:
        ref, nt = oracle_lib.trace(sc, rays, isect=isect, ties=True)
        w, c = oracle_lib.walk(b, rays, isect=isect)
        assert np.array_equal(ref["t"], w["t"])
        ok = nt <= 1
        assert np.array_equal(ref["prim"][ok], w["prim"][ok])
        assert np.array_equal(ref["u"][ok], w["u"][ok])
        assert np.array_equal(ref["v"][ok], w["v"][ok])
    return s


def test_product_bvh_prunes_exactly_soup(vsr, oracle_lib):
    sc = W.random_soup(2000, seed=81)
    rays = W.random_rays(4000, seed=82)
    o = oracle_lib
    _walker_vs_bruteforce(vsr, o, sc, rays, (o.DEFAULT, o.ALPHA_TEX, o.ALPHA_PROC))


def test_product_bvh_prunes_exactly_c1(vsr, oracle_lib):
    sc, rays = W.config("C1")
    o = oracle_lib
    for ml in (1, 2, 4):
        _walker_vs_bruteforce(vsr, o, sc, rays, (o.DEFAULT, o.ALPHA_TEX, o.ALPHA_PROC), ml)


@pytest.mark.slow
def test_product_bvh_prunes_exactly_c2_sample(vsr, oracle_lib):
    """C2 billboard forest (flat, thin boxes): walker over the product's padded
    BVH equals brute force on a seeded ray subsample."""
    texs = W.tree_textures(16, 256, 2)
    sc = W.forest_scene(textures=texs)
    rays = W.pinhole_rays((0.0, 4.0, -280.0), (0.0, 4.0, 0.0), (0.0, 1.0, 0.0), 45.0, 1920, 1080)
    idx = np.random.default_rng(5).choice(rays.n, 1024, replace=False)
    o = oracle_lib
    _walker_vs_bruteforce(vsr, o, sc, rays.data[idx], (o.DEFAULT, o.ALPHA_TEX))


def test_import_validation(vsr):
    sc = W.random_soup(200, seed=91)
    e = vsr.Scene.from_workload(sc, device=-1).build().export()
    bad = dict(e)
    bad["nodes"] = e["nodes"].copy()
    bad["nodes"][0, 12] = bad["nodes"][0, 13]        # two refs to the same subtree
    assert _err(vsr, lambda: vsr.Scene.import_arrays(bad)) == vsr.ERR_INVALID_ARG
    bad = dict(e)
    bad["sides"] = e["sides"].copy()
    bad["sides"][3, 6] = 10 ** 6                     # texel offset past the alpha plane
    assert _err(vsr, lambda: vsr.Scene.import_arrays(bad)) == vsr.ERR_INVALID_ARG
    bad = dict(e)
    bad["root_ref"] = 0x80000000 | (3 << 26) | 198   # leaf range past the end
    assert _err(vsr, lambda: vsr.Scene.import_arrays(bad)) == vsr.ERR_INVALID_ARG


def test_checkpoint_roundtrip(vsr, tmp_path):
    """checkpoint.save_scene / checkpoint.load_scene: a saved host-only scene re-imports (re-validated) to the
    identical export arrays; a corrupted file is rejected by the importer's validation."""
    from paper_1912_12786_b200 import checkpoint as io
    sc = W.random_soup(400, seed=81)
    s = vsr.Scene.from_workload(sc, device=-1).build()
    p = str(tmp_path / "s.npz")
    io.save_scene(s, p)
    t = io.load_scene(p, device=-1)
    a, b = s.export(), t.export()
    for k in ("nodes", "tris", "sides", "texdescs", "texels", "root_lo", "root_hi"):
        assert np.array_equal(a[k], b[k]), k
    assert a["root_ref"] == b["root_ref"]
    z = dict(np.load(p))
    z["nodes"] = z["nodes"].copy()
    z["nodes"][0, 12] = 10 ** 6            # an out-of-range child reference
    bad = str(tmp_path / "bad.npz")
    np.savez(bad, **z)
    with pytest.raises(vsr.VsrError):
        io.load_scene(bad, device=-1)
