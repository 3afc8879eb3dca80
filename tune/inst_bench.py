"""Instanced-forest (NEXT-2) and multi-hit timing for A/B builds: VSR_LIB=<lib> python
tune/inst_bench.py [reps].  CUDA events, L2 flushed (256 MiB read) before each launch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1912_12786_b200 import vsr  # noqa: E402


def timeit(fn, reps, flush, acc):
    for _ in range(3):
        torch.sum(flush, 0, out=acc)
        fn()
    ms = []
    for _ in range(reps):
        torch.sum(flush, 0, out=acc)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms))


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    torch.cuda.set_device(0)
    rays = W.rays_for("C2")
    d = torch.from_numpy(rays.data).cuda()
    n = rays.n
    flush = torch.zeros(64 << 20, device="cuda")
    acc = torch.zeros((), device="cuda")
    models, ibvh, imat = W.instanced_forest()
    sc = [vsr.Scene.from_workload(s).build() for s in models]
    inst = vsr.Instances(sc, ibvh, imat)
    hits = torch.empty((n, 4), device="cuda")
    ids = torch.empty((n,), dtype=torch.int32, device="cuda")
    out = {}
    for qn, q in (("any", vsr.ANY), ("closest", vsr.CLOSEST)):
        ms = timeit(lambda: inst.trace(d, q, vsr.ALPHA_TEXTURE, hits=hits, inst=ids), reps, flush, acc)
        out[f"instanced_{qn}"] = (round(n / ms / 1e3, 1), round(ms, 4))
    s = vsr.Scene.from_workload(W.scene("C2")).build()
    mh = torch.empty((n, 4, 4), device="cuda")
    mn = torch.empty((n,), dtype=torch.int32, device="cuda")
    ms = timeit(lambda: s.trace_multi(d, 4, vsr.ALPHA_TEXTURE, hits=mh, num_hits=mn), reps, flush, acc)
    out["multi4_any_alpha"] = (round(n / ms / 1e3, 1), round(ms, 4))
    print(os.environ.get("VSR_LIB", "default"), out)


if __name__ == "__main__":
    main()
