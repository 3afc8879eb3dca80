"""Small kernel workload for compute-sanitizer.

    compute-sanitizer --tool memcheck  python tools/sanitize_gpu.py [--quick]
    compute-sanitizer --tool racecheck python tools/sanitize_gpu.py --quick

Runs the trace kernels on C1 (every query x intersector, 4096 rays) and on a
64 Ki-ray subset of the C2 frame (ANY / CLOSEST with the alpha-texture, the
counting and the default intersectors, plus multi-hit, lists and instances),
so every kernel family of libvsr.so executes under the tool at least once.
It checks nothing itself (the parity tests do); its exit code and the tool's
report are the evidence.  One tool per gpurun call (B200_PROFILING.md).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1912_12786_b200 import vsr  # noqa: E402


def main():
    quick = "--quick" in sys.argv
    torch.cuda.set_device(0)
    kinds = [vsr.NONE, vsr.DEFAULT, vsr.ALPHA_TEXTURE, vsr.ALPHA_PROCEDURAL, vsr.COUNT,
             vsr.COUNT_ALPHA_TEXTURE, vsr.ALPHA_TEXTURE_BILINEAR, vsr.ALPHA_PROCEDURAL_UV]
    sc, rays = W.config("C1")
    s1 = vsr.Scene.from_workload(sc, device=0).build(max_leaf_size=1)
    d1 = torch.from_numpy(rays.data).cuda()
    for q in (vsr.CLOSEST, vsr.ANY):
        for k in kinds:
            s1.trace(d1, query=q, isect=k)
    s1.trace_multi(d1, 4, vsr.ALPHA_TEXTURE)
    torch.cuda.synchronize()
    print("C1 done", flush=True)

    sc2 = W.scene("C2")
    r2 = W.rays_for("C2")
    n = 8192 if quick else 65536
    rng = np.random.default_rng(5)
    sub = np.ascontiguousarray(r2.data[np.sort(rng.choice(r2.n, n, replace=False))])
    s2 = vsr.Scene.from_workload(sc2, device=0).build()
    d2 = torch.from_numpy(sub).cuda()
    for q in (vsr.CLOSEST, vsr.ANY):
        for k in (vsr.DEFAULT, vsr.ALPHA_TEXTURE, vsr.COUNT_ALPHA_TEXTURE):
            s2.trace(d2, query=q, isect=k)
    s2.trace_multi(d2, 4, vsr.ALPHA_TEXTURE)
    torch.cuda.synchronize()
    print("C2 subset done", flush=True)
    if quick:
        return
    parts = [vsr.Scene.from_workload(p, device=0).build() for p in W.split_scene(sc2, 3)]
    g = vsr.Group(parts)
    for q in (vsr.CLOSEST, vsr.ANY):
        g.trace(d2, query=q, isect=vsr.ALPHA_TEXTURE)
    models, ibvh, imat = W.instanced_forest(n_instances=500)
    iscenes = [vsr.Scene.from_workload(s, device=0).build() for s in models]
    inst = vsr.Instances(iscenes, ibvh, imat)
    for q in (vsr.CLOSEST, vsr.ANY):
        inst.trace(d2, query=q, isect=vsr.ALPHA_TEXTURE)
    s3 = vsr.Scene.from_workload(sc2, device=0)
    s3.build_gpu(2)
    s3.trace(d2, query=vsr.ANY, isect=vsr.ALPHA_TEXTURE)
    torch.cuda.synchronize()
    print("compounds + GPU builder done", flush=True)


if __name__ == "__main__":
    main()
