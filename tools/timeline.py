"""Diagnostic: per-warp (SM, start, end) timeline of the C2 headline trace.

    VSR_LIB=variants/lib_timeline.so QUERY=any python tools/timeline.py

(the variant is built with -DVSR_TIMELINE; the kernel then stores per-warp SM id and global-timer
start/end in the counts buffer).  Prints the launch span, the per-SM first start / last end, the
time SMs sit idle before the span ends (tail) and warp-duration percentiles."""
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
q = vsr.ANY if os.environ.get("QUERY", "any") == "any" else vsr.CLOSEST
flush = torch.zeros(64 << 20, device="cuda")
for _ in range(5):
    flush.sum()
    # raw call: the diagnostic build writes one record per WARP into the counts buffer
    s.trace_raw(d.data_ptr(), rays.n, q, isect, hits.data_ptr(), tl.data_ptr(),
                torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
out = tl.cpu().numpy().view(np.uint32)[: rays.n // 32]
np.save(os.environ.get("OUT", "gpurun_out/timeline.npy"), out)
sm = out[:, 0].astype(np.int64)
t0 = (out[:, 3].astype(np.int64) << 32) | out[:, 1].astype(np.int64)
t1 = (t0 & ~0xFFFFFFFF) | out[:, 2].astype(np.int64)
t1 = np.where(t1 < t0, t1 + (1 << 32), t1)
base = t0.min()
t0, t1 = (t0 - base) / 1e3, (t1 - base) / 1e3          # µs
span = t1.max()
first = np.array([t0[sm == k].min() for k in np.unique(sm)])
last = np.array([t1[sm == k].max() for k in np.unique(sm)])
dur = t1 - t0
busy = np.zeros(len(np.unique(sm)))
print(f"span {span:.1f} us over {len(first)} SMs, {len(t0)} warps")
print(f"per-SM first start: min {first.min():.2f} median {np.median(first):.2f} max {first.max():.2f} us")
print(f"per-SM last end:    min {last.min():.1f} median {np.median(last):.1f} max {last.max():.1f} us")
print(f"mean SM idle at the tail: {np.mean(span - last):.1f} us ({100 * np.mean(span - last) / span:.1f} %)")
for p in (50, 90, 99, 99.9, 100):
    print(f"warp duration p{p}: {np.percentile(dur, p):.1f} us")
late = t0 > 0.9 * span
print(f"warps starting in the last 10 % of the span: {late.sum()}, their mean duration {dur[late].mean() if late.any() else 0:.1f} us")
# the critical path: the warps that end last — when did they start, how long did they run
order = np.argsort(-t1)[:10]
print("last-ending warps (start us, duration us, warp id):")
for w in order:
    print(f"  {t0[w]:7.1f} {dur[w]:7.1f} {w}")
slow = np.argsort(-dur)[:10]
print("slowest warps (start us, duration us, end us):")
for w in slow:
    print(f"  {t0[w]:7.1f} {dur[w]:7.1f} {t1[w]:7.1f}")
print(f"lower bound from the slowest warp: {dur.max():.1f} us of the {span:.1f} us span")
