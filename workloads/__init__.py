"""Seeded synthetic workload generators shared by the oracle tests, the CUDA
parity tests and ``bench.py``.

This module holds *inputs only*: scene geometry, alpha textures and camera
rays shaped like the paper's use cases (PAPER.md:4-20 [Fig. 1 teaser],
PAPER.md:282-322 [§4 use cases]).  It contains none of the method's
arithmetic — no ray/triangle test, no slab test, no texture lookup, no
traversal — so that neither the oracle (``oracle/``) nor the product
(``paper_1912_12786_b200``) can borrow from the other through it.

Recipes follow SURVEY.md §8(d) (configs C1–C5) and are restated in
DESIGN.md §"Input recipe".
"""
from .gen import (  # noqa: F401
    Scene,
    Rays,
    pcg_hash,
    quad_pair_scene,
    quad_pair_rays,
    tree_textures,
    stress_textures,
    forest_scene,
    heightfield_scene,
    c4_scene,
    c5_scene,
    pinhole_rays,
    config,
    scene,
    rays_for,
    CAMERAS,
    CONFIGS,
    random_soup,
    random_rays,
    stacked_quads,
    split_scene,
    concat_scenes,
    tree_model,
    object_from_world,
    instanced_forest,
)
