"""Diagnose direct vs warp schedule differences on the ragged-test inputs."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_12786_b200 import vsr as V
import workloads as W
import oracle as o
from tests import bvh_check
o.build()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
sc = W.random_soup(2000, seed=900 + n)
rays = W.random_rays(n, seed=901 + n).data
s = V.Scene.from_workload(sc).build()
b = bvh_check.to_oracle(s.export())
def run(q, k, env):
    old = {}
    for kk, vv in env.items():
        old[kk] = os.environ.get(kk); os.environ[kk] = vv
    r = torch.from_numpy(np.ascontiguousarray(rays, np.float32)).cuda()
    h, c = s.trace(r, query=q, isect=k)
    torch.cuda.synchronize()
    for kk, vv in old.items():
        if vv is None: del os.environ[kk]
        else: os.environ[kk] = vv
    return V.hits_to_numpy(h), (V.counts_to_numpy(c) if c is not None else None)
for q, oq in ((V.CLOSEST, o.CLOSEST), (V.ANY, o.ANY)):
    for k, ok in ((V.COUNT_ALPHA_TEXTURE, o.ALPHA_TEX), (V.ALPHA_TEXTURE, o.ALPHA_TEX), (V.DEFAULT, o.DEFAULT)):
        wh, wc = o.walk(b, rays, oq, ok)
        res = {}
        for name, env in (("direct", {}), ("warp", {"VSR_SCHED": "warp"}), ("noorder", {"VSR_ORDER": "0"}),
                          ("warp_noorder", {"VSR_SCHED": "warp", "VSR_ORDER": "0"}), ("region", {"VSR_SCHED": "region"})):
            h, c = run(q, k, env)
            dh = np.nonzero((h.view(np.uint32).reshape(n, 4) != wh.view(np.uint32).reshape(n, 4)).any(1))[0]
            msg = f"q={q} k={k} {name:13s} hit-diff vs walker: {dh.size}"
            if c is not None and k == V.COUNT_ALPHA_TEXTURE:
                dc = np.nonzero((c["boxes"] != wc["boxes"]) | (c["tris"] != wc["tris"]))[0]
                msg += f" count-diff: {dc.size}"
            if dh.size:
                i = dh[0]
                msg += f" first ray {i} gpu {h[i]} walker {wh[i]}"
            print(msg, flush=True)
