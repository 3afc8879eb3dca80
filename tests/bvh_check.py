"""Independent structural validator for BVHs in the export layout (DESIGN.md
§"Data layout"), used on both the oracle's and the product's trees.  Written
from the documented layout, sharing nothing with either builder."""
import numpy as np

LEAF = 0x80000000


def as_dict(b):
    if isinstance(b, dict):
        return b
    return {"root_ref": b.root_ref, "root_lo": b.root_lo, "root_hi": b.root_hi, "nodes": b.nodes,
            "tris": b.tris, "sides": b.sides, "texdescs": b.texdescs, "texels": b.texels}


def to_oracle(b):
    """Export dict -> oracle.BvhArrays (for walker C)."""
    import oracle
    if not isinstance(b, dict):
        return b
    return oracle.BvhArrays(int(b["root_ref"]), np.asarray(b["root_lo"], np.float32),
                            np.asarray(b["root_hi"], np.float32), b["nodes"], b["tris"], b["sides"],
                            b["texdescs"], b["texels"])


def validate(b, vertices=None, max_leaf=None, slack=1e-5):
    """Check: tree shape, every triangle in exactly one leaf, boxes contain
    their subtrees, leaf sizes, depth <= 64, triangles reproduce the caller's
    vertices (v0 exact, e1/e2 = fl(v1-v0), fl(v2-v0)).  Returns max depth."""
    b = as_dict(b)
    nodes = np.asarray(b["nodes"], np.uint32)
    tris = np.asarray(b["tris"], np.uint32)
    nf = nodes.view(np.float32)
    tf = tris.view(np.float32)
    v0 = tf[:, 0:3]
    e1 = tf[:, 4:7]
    e2 = tf[:, 8:11]
    tlo = np.minimum(np.minimum(v0, v0 + e1), v0 + e2)
    thi = np.maximum(np.maximum(v0, v0 + e1), v0 + e2)
    seen_tri = np.zeros(tris.shape[0], np.int64)
    seen_node = np.zeros(nodes.shape[0], np.int64)
    max_depth = 0
    stack = [(int(b["root_ref"]), np.asarray(b["root_lo"]), np.asarray(b["root_hi"]), 0)]
    while stack:
        ref, lo, hi, depth = stack.pop()
        assert depth <= 64, "deeper than the 64-entry stack"
        max_depth = max(max_depth, depth)
        if ref & LEAF:
            first = ref & 0x03FFFFFF
            cnt = ((ref >> 26) & 31) + 1
            if max_leaf is not None:
                assert cnt <= max_leaf
            assert first + cnt <= tris.shape[0]
            sl = slice(first, first + cnt)
            seen_tri[sl] += 1
            assert np.all(tlo[sl] >= lo - slack * np.maximum(1, np.abs(lo)))
            assert np.all(thi[sl] <= hi + slack * np.maximum(1, np.abs(hi)))
            continue
        assert 0 <= ref < nodes.shape[0]
        seen_node[ref] += 1
        for c in range(2):
            # per axis k the node stores (lo0.k, lo1.k, hi0.k, hi1.k)
            clo = nf[ref, [0 + c, 4 + c, 8 + c]]
            chi = nf[ref, [2 + c, 6 + c, 10 + c]]
            assert np.all(clo <= chi)
            assert np.all(clo >= lo - slack * np.maximum(1, np.abs(lo)))
            assert np.all(chi <= hi + slack * np.maximum(1, np.abs(hi)))
            stack.append((int(nodes[ref, 12 + c]), clo, chi, depth + 1))
    assert np.all(seen_tri == 1), "every triangle in exactly one leaf"
    assert np.all(seen_node == 1), "every node reachable exactly once"
    prim = tris[:, 3]
    assert len(np.unique(prim)) == prim.shape[0]
    if vertices is not None:
        vt = np.asarray(vertices, np.float32)[prim]
        assert np.array_equal(v0, vt[:, 0:3])
        assert np.array_equal(e1, (vt[:, 3:6] - vt[:, 0:3]).astype(np.float32))
        assert np.array_equal(e2, (vt[:, 6:9] - vt[:, 0:3]).astype(np.float32))
    return max_depth
