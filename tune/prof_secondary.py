"""Probe run for ncu captures of the secondary kernels:
the instanced forest (trace_instances_kernel) and the multi-hit query k = 4
(trace_multi_kernel) on the C2 camera, ANY / CLOSEST + alpha texture, 3 launches
each with an L2 flush before each.

    python tune/prof_secondary.py [instances|multi|both]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1912_12786_b200 import vsr  # noqa: E402


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "both"
    q = vsr.ANY if "--closest" not in sys.argv else vsr.CLOSEST
    torch.cuda.set_device(0)
    rays = W.rays_for("C2")
    d = torch.from_numpy(rays.data).cuda()
    flush = torch.zeros(64 << 20, device="cuda")
    acc = torch.zeros((), device="cuda")
    if what in ("instances", "both"):
        models, ibvh, imat = W.instanced_forest()
        sc = [vsr.Scene.from_workload(s).build() for s in models]
        inst = vsr.Instances(sc, ibvh, imat)
        for _ in range(3):
            torch.sum(flush, 0, out=acc)
            inst.trace(d, q, vsr.ALPHA_TEXTURE)
        torch.cuda.synchronize()
    if what in ("multi", "both"):
        s = vsr.Scene.from_workload(W.scene("C2")).build()
        for _ in range(3):
            torch.sum(flush, 0, out=acc)
            s.trace_multi(d, 4, vsr.ALPHA_TEXTURE)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
