"""Parity report (run on a B200): CUDA path vs oracle S / walker C on every config.

For each config x query x intersector it records rays compared, hits, exact fp32 ties,
the oracle's ambiguity classes X1-X4 (double shadow), and mismatches
after the tie rule (must be 0), plus whether t/u/v were bit-exact.  Counts: bit-exact
fraction against walker C.  Output: JSON on stdout (commit it under profiles/).

    python tools/parity_report.py > profiles/r02_parity_report.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: this is a test tool)
import workloads as W  # noqa: E402
from paper_1912_12786_b200 import vsr  # noqa: E402
from tests import bvh_check  # noqa: E402

MISS = 0xFFFFFFFF
KINDS = [("none", vsr.NONE, oracle.NONE), ("default", vsr.DEFAULT, oracle.DEFAULT),
         ("alpha_texture", vsr.ALPHA_TEXTURE, oracle.ALPHA_TEX),
         ("alpha_procedural", vsr.ALPHA_PROCEDURAL, oracle.ALPHA_PROC)]
QUERIES = [("closest", vsr.CLOSEST, oracle.CLOSEST), ("any", vsr.ANY, oracle.ANY)]


def compare(sc, rays, q, oq, ok, g, ref, fl, nt):
    n = rays.shape[0]
    g_hit = g["prim"] != MISS
    r_hit = ref["prim"] != MISS
    flag_miss = int(np.sum(g_hit != r_hit))
    bad = flag_miss
    ties = 0
    exact = True
    if oq == oracle.CLOSEST:
        diff = np.nonzero((g["prim"] != ref["prim"]) & g_hit & r_hit)[0]
        if diff.size:
            acc, e = oracle.eval_pairs(sc, rays[diff], g["prim"][diff], ok)
            tie = (nt[diff] > 1) & acc & (e["t"] == ref["t"][diff]) & (e["t"] == g["t"][diff])
            ties = int(tie.sum())
            bad += int((~tie).sum())
        same = (g["prim"] == ref["prim"]) & g_hit
        exact = bool(np.all((g["t"][same] == ref["t"][same]) & (g["u"][same] == ref["u"][same])
                            & (g["v"][same] == ref["v"][same])))
    else:   # every returned any-hit validated
        idx = np.nonzero(g_hit)[0]
        acc, e = oracle.eval_pairs(sc, rays[idx], g["prim"][idx], ok)
        bad += int((~acc).sum())
        gi = g[idx]
        exact = bool(np.all(~acc | ((e["t"] == gi["t"]) & (e["u"] == gi["u"]) & (e["v"] == gi["v"]))))
    return {"rays": int(n), "hits": int(g_hit.sum()), "exact_ties": ties, "mismatches": int(bad),
            "tuv_bit_exact": exact,
            "X1_near_tie": int(np.sum(fl & oracle.X1 != 0)), "X2_edge_graze": int(np.sum(fl & oracle.X2 != 0)),
            "X3_texel_edge": int(np.sum(fl & oracle.X3 != 0)), "X4_checker_edge": int(np.sum(fl & oracle.X4 != 0)),
            "X5_alpha_near": int(np.sum(fl & oracle.X5 != 0))}


def run_config(name, sample, textures, kinds=None):
    sc, rays = W.scene(name, textures), W.rays_for(name)
    s = vsr.Scene.from_workload(sc).build()
    d = torch.from_numpy(rays.data).cuda()
    osc = oracle.OracleScene(sc)
    idx = (np.arange(rays.n) if sample is None or sample >= rays.n
           else np.sort(np.random.default_rng(2024).choice(rays.n, sample, replace=False)))
    sub = rays.data[idx]
    out = {"config": name, "rays_in_launch": rays.n, "rays_compared": int(len(idx)),
           "triangles": sc.num_tris, "results": {}}
    for qn, q, oq in QUERIES:
        for kn, k, ok in (kinds or KINDS):
            hits, _ = s.trace(d, q, k)
            torch.cuda.synchronize()
            g = vsr.hits_to_numpy(hits)[idx]
            ref, fl, nt = oracle.trace(osc, sub, query=oq, isect=ok, flags=True, ties=True)
            out["results"][f"{qn}/{kn}"] = compare(osc, sub, q, oq, ok, g, ref, fl, nt)
    # counts: full launch vs walker C on the exported BVH (a bounded ray sample for C5)
    b = bvh_check.to_oracle(s.export())
    cidx = np.arange(rays.n) if rays.n <= 4_200_000 else \
        np.sort(np.random.default_rng(7).choice(rays.n, 1 << 20, replace=False))
    for kn, k, ok in (("count", vsr.COUNT, oracle.DEFAULT),
                      ("count_alpha_texture", vsr.COUNT_ALPHA_TEXTURE, oracle.ALPHA_TEX)):
        hits, counts = s.trace(d, vsr.CLOSEST, k)
        torch.cuda.synchronize()
        c = vsr.counts_to_numpy(counts)[cidx]
        h = vsr.hits_to_numpy(hits)[cidx]
        wh, wc = oracle.walk(b, rays.data[cidx], isect=ok)
        out["results"][f"closest/{kn}"] = {
            "rays": int(len(cidx)),
            "counts_bit_exact": bool(np.array_equal(c["boxes"], wc["boxes"]) and
                                     np.array_equal(c["tris"], wc["tris"]) and
                                     np.array_equal(c["alpha"], wc["alpha"])),
            "hits_bit_exact_vs_walker": bool(h.tobytes() == wh.tobytes()),
            "mean_boxes": float(c["boxes"].mean()), "mean_tris": float(c["tris"].mean())}
    s.close()
    return out


def main():
    t0 = time.time()
    textures = W.tree_textures(16, 1024, 2)
    # C2: the full 2,073,600-ray frame for the headline intersectors; C4 / C5: 16,384-ray
    # seeded samples of the full launches (oracle S is brute force over 1.04 M / 10.2 M tris)
    head = [k for k in KINDS if k[0] in ("default", "alpha_texture")]
    plan = [("C1", None, None), ("C2", None, head), ("C2", 65536, None), ("C4", 16384, None),
            ("C5", 16384, head)]
    if "--quick" in sys.argv:
        plan = [("C1", None, None), ("C2", 8192, None)]
    rep = {"device": torch.cuda.get_device_name(0), "configs": []}
    for name, sample, kinds in plan:
        rep["configs"].append(run_config(name, sample, textures, kinds))
        print(f"{name} done {time.time() - t0:.1f}s", file=sys.stderr)
    tot = sum(r["mismatches"] for c in rep["configs"] for r in c["results"].values() if "mismatches" in r)
    rep["total_mismatches"] = tot
    rep["all_counts_bit_exact"] = all(r.get("counts_bit_exact", True) for c in rep["configs"]
                                      for r in c["results"].values())
    print(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
