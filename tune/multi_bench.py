"""Median time of the multi-hit query (k = 4, ANY-independent: the 4 nearest accepted hits,
alpha texture) on C2, CUDA events, L2 flushed before each launch.
    python tune/multi_bench.py [iters]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1912_12786_b200 import vsr  # noqa: E402

it = int(sys.argv[1]) if len(sys.argv) > 1 else 50
torch.cuda.set_device(0)
rays = W.rays_for("C2")
d = torch.from_numpy(rays.data).cuda()
n = d.shape[0]
s = vsr.Scene.from_workload(W.scene("C2")).build()
hits = torch.empty((n, 4, 4), dtype=torch.float32, device="cuda")
nh = torch.empty((n,), dtype=torch.int32, device="cuda")
flush = torch.zeros(64 << 20, device="cuda")
acc = torch.zeros((), device="cuda")
ts = []
for i in range(it + 5):
    torch.sum(flush, 0, out=acc)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s.trace_multi(d, 4, vsr.ALPHA_TEXTURE, hits=hits, num_hits=nh)
    b.record()
    torch.cuda.synchronize()
    if i >= 5:
        ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
print(f"multi k=4 alpha C2: {ms:.4f} ms {n / ms / 1e6:.1f} Grays/s")
