"""Parity comparison between the CUDA path and oracle S.

Bar (north_star + DESIGN.md "Tolerances"): hit/miss and prim_id bit-exact,
except exact fp32 ties in t, where any tied candidate is correct (checked for
validity); t within 1e-5 relative and u, v within 1e-5 absolute — the
contract actually delivers bit-exact t/u/v, which is asserted separately
(``exact=True``); any-hit: hit flag exact, returned prim must be in the
accepted set with the oracle's (t, u, v) for that prim.
"""
import numpy as np

MISS = 0xFFFFFFFF


def compare(oracle, scene, rays, query, isect, gpu, ref, ntie=None, exact=True,
            alpha_threshold=0.01, checker_freq=8, max_report=5):
    """Return a dict summary; raise AssertionError on any out-of-tolerance ray."""
    rays = np.asarray(getattr(rays, "data", rays), np.float32).reshape(-1, 8)
    g_hit = gpu["prim"] != MISS
    r_hit = ref["prim"] != MISS
    bad = []
    assert np.array_equal(g_hit, r_hit), _report("hit/miss", np.nonzero(g_hit != r_hit)[0],
                                                 gpu, ref, max_report)
    n_ties = 0
    if query == oracle.CLOSEST:
        same = gpu["prim"] == ref["prim"]
        diff = np.nonzero(~same)[0]
        if diff.size:
            # only legitimate reason: an exact tie in t among accepted candidates
            assert ntie is not None and np.all(ntie[diff] > 1), _report(
                "prim", diff[ntie[diff] <= 1] if ntie is not None else diff, gpu, ref, max_report)
            acc, e = oracle.eval_pairs(scene, rays[diff], gpu["prim"][diff], isect,
                                       alpha_threshold, checker_freq)
            ok = acc & (e["t"] == ref["t"][diff]) & (e["t"] == gpu["t"][diff]) & \
                (e["u"] == gpu["u"][diff]) & (e["v"] == gpu["v"][diff])
            assert np.all(ok), f"invalid tie winner rays {diff[~ok][:max_report]}"
            n_ties = int(diff.size)
        s = same & g_hit
        _check_tuv(gpu, ref, s, exact)
    else:
        # every returned any-hit: the prim must be in the accepted set A, with the oracle's
        # (t, u, v) for that prim (several answers are correct)
        idx = np.nonzero(g_hit)[0]
        acc, e = oracle.eval_pairs(scene, rays[idx], gpu["prim"][idx], isect, alpha_threshold,
                                   checker_freq)
        g = gpu[idx]
        if exact:
            ok = acc & (e["t"] == g["t"]) & (e["u"] == g["u"]) & (e["v"] == g["v"])
        else:
            ok = acc & (np.abs(e["t"] - g["t"]) <= 1e-5 * np.abs(e["t"])) & \
                (np.abs(e["u"] - g["u"]) <= 1e-5) & (np.abs(e["v"] - g["v"]) <= 1e-5)
        bad = list(idx[~ok])
        assert not bad, _report("any-hit prim not in accepted set", bad, gpu, ref, max_report)
    miss = ~g_hit
    assert np.all(gpu["t"][miss] == np.inf) and np.all(gpu["u"][miss] == 0) \
        and np.all(gpu["v"][miss] == 0), "miss record must be (inf, 0, 0, ~0)"
    return {"rays": int(rays.shape[0]), "hits": int(g_hit.sum()), "exact_ties": n_ties}


def _check_tuv(gpu, ref, mask, exact):
    if exact:
        bad = np.nonzero(mask & ((gpu["t"] != ref["t"]) | (gpu["u"] != ref["u"]) |
                                 (gpu["v"] != ref["v"])))[0]
        assert bad.size == 0, _report("t/u/v not bit-exact", bad, gpu, ref, 5)
    else:
        dt = np.abs(gpu["t"][mask] - ref["t"][mask]) <= 1e-5 * np.abs(ref["t"][mask])
        du = np.abs(gpu["u"][mask] - ref["u"][mask]) <= 1e-5
        dv = np.abs(gpu["v"][mask] - ref["v"][mask]) <= 1e-5
        assert np.all(dt & du & dv), "t/u/v outside tolerance"


def _report(what, idx, gpu, ref, k):
    idx = list(idx)[:k]
    rows = [f"  ray {i}: gpu={tuple(gpu[i])} ref={tuple(ref[i])}" for i in idx]
    return f"{what}: {len(list(idx))}+ rays differ\n" + "\n".join(rows)
