"""Diagnostic: per-warp (SM, start, end) timeline of the C2 headline trace.

Run with VSR_LIB=variants/lib_timeline.so (built with -DVSR_TIMELINE)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1912_12786_b200 import vsr  # noqa: E402

sc, rays = W.config("C2")
s = vsr.Scene.from_workload(sc).build()
d = torch.from_numpy(rays.data).cuda()
hits = torch.empty((rays.n, 4), device="cuda")
tl = torch.zeros((rays.n // 32 + 1, 4), dtype=torch.int32, device="cuda")
isect = getattr(vsr, os.environ.get("ISECT", "ALPHA_TEXTURE"))
for _ in range(5):
    s.trace(d, vsr.CLOSEST, isect, hits=hits, counts=tl)
torch.cuda.synchronize()
out = tl.cpu().numpy().view(np.uint32)
np.save(os.environ.get("OUT", "gpurun_out/timeline.npy"), out)
print("saved", out.shape)
