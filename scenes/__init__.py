"""Seeded synthetic scene generators shared by the oracle tests, the GPU tests and bench.py.

This module draws inputs only.  It contains none of the method's arithmetic
(no warp radius, no Kalman predict, no stamping test, no relaxation): it
produces the *inputs* the paper's planner consumes (grid, static walls, robot
pose, goal cell, Kalman tracks, configuration), so that the CPU oracle
(`oracle/`) and the CUDA path (`paper_1903_07441_b200/`) can be fed the same
bytes while sharing no code.
"""
from .gen import (  # noqa: F401
    Scene,
    WarpCfg,
    default_warp_cfg,
    scene_c1,
    scene_random,
    scene_c2,
    scene_c3,
    scene_c4,
    scene_c5,
    advance_scene,
    detections,
    SimCfg,
    scene_sim,
    annulus_fixed,
    random_small_map,
    CONFIGS,
)
