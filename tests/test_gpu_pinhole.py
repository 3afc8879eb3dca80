"""Fused primary-ray generation (vsr_trace_pinhole): the in-kernel rays
equal the input recipe's host rays bit for bit, shown by hits (t, u, v, prim) and counts
bit-exact against vsr_trace on workloads.pinhole_rays for the same camera."""
import numpy as np
import pytest

import workloads as W

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


@pytest.mark.parametrize("res,spp", [((480, 272), 1), ((128, 64), 4), ((64, 32), 9)])
def test_pinhole_equals_host_rays(V, res, spp):
    eye, look, up, fov, _, _, _ = W.CAMERAS["C2"]
    w, h = res
    sc = W.scene("C2")
    scene = V.Scene.from_workload(sc).build()
    rays = W.pinhole_rays(eye, look, up, fov, w, h, spp)
    cam = V.pinhole_camera(eye, look, up, fov, w, h, spp)
    d_rays = torch.from_numpy(rays.data).cuda()
    for q in (V.CLOSEST, V.ANY):
        for k in (V.NONE, V.ALPHA_TEXTURE, V.ALPHA_PROCEDURAL, V.COUNT_ALPHA_TEXTURE):
            h1, c1 = scene.trace(d_rays, q, k)
            h2, c2 = scene.trace_pinhole(cam, q, k)
            torch.cuda.synchronize()
            assert torch.equal(h1.view(torch.int32), h2.view(torch.int32)), (q, k)
            if c1 is not None:
                assert torch.equal(c1, c2)
    assert (V.hits_to_numpy(h2)["prim"] != 0xFFFFFFFF).mean() > 0.05


def test_pinhole_validation(V):
    scene = V.Scene.from_workload(W.random_soup(50, seed=1)).build()
    bad = V.pinhole_camera((0, 0, -5), (0, 0, 0), (0, 1, 0), 45.0, 60, 64)   # width % 8
    with pytest.raises(V.VsrError):
        scene.trace_pinhole(bad)
    bad = V.pinhole_camera((0, 0, -5), (0, 0, 0), (0, 1, 0), 45.0, 64, 64, spp=3)
    with pytest.raises(V.VsrError):
        scene.trace_pinhole(bad)
    cam = V.pinhole_camera((0, 0, -5), (0, 0, 0), (0, 1, 0), 45.0, 64, 64)
    with pytest.raises(V.VsrError):
        scene.trace_pinhole(cam, V.CLOSEST, V.RUNTIME_SWITCH_DEFAULT)


def test_c_program_traces_on_the_gpu(V, tmp_path):
    """examples/c_trace_host.c: the whole path (create, build, vsr_trace_host with the alpha
    intersector) driven from plain C."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.dirname(V.LIB_PATH)
    exe = tmp_path / "vsr_ct"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-I", os.path.join(root, "include"),
                    os.path.join(root, "examples", "c_trace_host.c"), "-L", libdir, "-lvsr",
                    f"-Wl,-rpath,{libdir}", "-lm", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr


def test_checkpoint_restores_a_traceable_scene(V, tmp_path):
    """A scene saved with checkpoint.save_scene and restored on the GPU traces bit-identically."""
    from paper_1912_12786_b200 import checkpoint
    sc, rays = W.config("C2", 128, 64)
    s = V.Scene.from_workload(sc).build()
    p = str(tmp_path / "c2.npz")
    checkpoint.save_scene(s, p)
    t = checkpoint.load_scene(p, device=0)
    d = torch.from_numpy(rays.data).cuda()
    for q in (V.CLOSEST, V.ANY):
        a, _ = s.trace(d, q, V.ALPHA_TEXTURE)
        b, _ = t.trace(d, q, V.ALPHA_TEXTURE)
        torch.cuda.synchronize()
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))
