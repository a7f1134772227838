"""B200-native hot path of the Time-Warped Grid planner (arXiv 1903.07441).

The compute path is libtwg.so (hand-written sm_100a CUDA behind the C ABI of
include/twg.h); :mod:`.twg` is its ctypes binding.  Nothing here imports the
CPU oracle.
"""
from .twg import (  # noqa: F401
    Planner,
    TwgError,
    lib,
    warp_cfg,
    relax_cfg,
    band_cfg,
    tracker_cfg,
    sim_cfg,
    tracks_array,
    LIB_PATH,
)
