import sys, numpy as np, torch
sys.path.insert(0, '.')
import workloads as W
from paper_1912_12786_b200 import vsr
for cfg in ("C2", "C4"):
    sc, rays = W.config(cfg)
    d = torch.from_numpy(rays.data).cuda()
    hits = torch.empty((rays.n, 4), device="cuda")
    flush = torch.zeros(64 << 20, device="cuda")
    for r in (4, 16, 64, 256):
        s = vsr.Scene.from_workload(sc).build_ploc(2, r)
        s.build_ploc(2, r)
        st = s.stats()
        ts = []
        for it in range(15):
            flush.sum()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); s.trace(d, vsr.ANY, vsr.ALPHA_TEXTURE, hits=hits); b.record(); b.synchronize()
            if it >= 5: ts.append(a.elapsed_time(b))
        print(cfg, "r", r, "build_ms %.1f" % st["build_ms"], "trace ms %.4f" % np.mean(ts), "depth", st["max_depth"], flush=True)
