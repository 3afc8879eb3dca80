"""Time the list query (vsr_trace_group) on C2 split into k sub-scenes: python tune/list_bench.py [k]"""
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_1912_12786_b200 import vsr  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
sc, rays = W.config("C2")
scenes = [vsr.Scene.from_workload(s).build() for s in W.split_scene(sc, k, axis=2)]
g = vsr.Group(scenes)
r = torch.from_numpy(rays.data).cuda()
flush = torch.zeros(64 << 20, device="cuda")
acc = torch.zeros((), device="cuda")
for q, name in ((vsr.ANY, "any"), (vsr.CLOSEST, "closest")):
    hits = torch.empty((rays.n, 4), device="cuda")
    which = torch.empty((rays.n,), dtype=torch.int32, device="cuda")
    ts = []
    for i in range(55):
        torch.sum(flush, 0, out=acc)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.trace(r, q, vsr.ALPHA_TEXTURE, hits=hits, which=which)
        b.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    print(f"list k={k} {name}: {ms:.4f} ms  {rays.n / ms / 1e3:.0f} Mrays/s")
