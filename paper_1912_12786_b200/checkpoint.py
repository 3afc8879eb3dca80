"""Checkpoint / resume of built acceleration structures (SURVEY.md §5 "checkpoint/resume").

A built scene is saved as its export-layout arrays (vsr_bvh_export: pair nodes, triangles,
sidecars, texture descriptors, the A8 alpha plane, root) in one `.npz`, and restored with
vsr_scene_import — which re-validates the whole structure — onto any device (or host-only,
device -1).  C5's 7.5 s host build becomes a file read.  No tracing arithmetic here.
"""
from __future__ import annotations

import numpy as np

from . import vsr

FORMAT = "vsr-bvh-export-v1"


def save_scene(scene: "vsr.Scene", path: str) -> None:
    arrs = scene.export()
    np.savez(path, format=np.array(FORMAT), abi=np.array(vsr.lib().vsr_abi_version()),
             root_ref=np.array(arrs["root_ref"], np.uint32), root_lo=arrs["root_lo"],
             root_hi=arrs["root_hi"], nodes=arrs["nodes"], tris=arrs["tris"], sides=arrs["sides"],
             texdescs=arrs["texdescs"], texels=arrs["texels"])


def load_scene(path: str, device: int = 0) -> "vsr.Scene":
    with np.load(path, allow_pickle=False) as z:
        if str(z["format"]) != FORMAT:
            raise ValueError(f"{path}: not a {FORMAT} file")
        if "abi" not in z or int(z["abi"]) != int(vsr.lib().vsr_abi_version()):
            # the export layout (nodes, sidecars) is versioned by the ABI number
            raise ValueError(f"{path}: written by ABI {int(z['abi']) if 'abi' in z else '?'}, "
                             f"this library is ABI {int(vsr.lib().vsr_abi_version())}")
        arrs = {k: z[k] for k in ("nodes", "tris", "sides", "texdescs", "texels", "root_lo",
                                  "root_hi")}
        arrs["root_ref"] = int(z["root_ref"])
    return vsr.Scene.import_arrays(arrs, device=device)
