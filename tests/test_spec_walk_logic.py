"""CPU check of the speculative-walk argument (row a7): with markers on ANY set of
distinct cells, a walker from the robot cell plus one walker per marker -- each stopping at the goal,
an obstacle, a cell without an in-grid neighbour, max_len, or the first marker it reaches -- chained
marker by marker (a marker reached twice = a cycle = no path; more than max_len cells = no path)
give exactly the single descent walk of Alg. 1 P:705 (oracle.walk).

This is the rule k_walk / k_spec_stitch implement on the GPU; here it is written in Python over the
oracle's index matrix M_idx (orc_index_matrix, pinned by P17) and compared with orc_walk (pinned by
P11), on converged, unconverged and cyclic fields.  No GPU and no CUDA-path data involved."""
import numpy as np
import pytest

import oracle
from scenes import random_small_map

MOVES = {0: (1, 0), 1: (-1, 0), 2: (0, 1), 3: (0, -1)}  # M_idx codes; 4 goal, 5 obstacle, 6 none


def _segment(m, start, markers, max_len, first_step_from=None):
    """One walker: cells after `start` until a terminal, a marker, or max_len (counted from start).
    Returns (state, cells, next_marker): state 1 goal, 2 no path, 3 marker."""
    x, y = start
    n, cells = 1, []
    code = m[y, x] if first_step_from is None else first_step_from
    while True:
        if code == 4:
            return 1, cells, None
        if code >= 5:
            return 2, cells, None
        if n + 1 > max_len:
            return 2, cells, None
        dx, dy = MOVES[int(code)]
        x, y = x + dx, y + dy
        cells.append((x, y))
        n += 1
        if (x, y) in markers:
            return 3, cells, markers[(x, y)]
        code = m[y, x]


def spec_walk(m, start, markers_list, max_len):
    """Walker 0 from start; walker k from marker k (first step from the marker's own code); chain."""
    markers = {c: k for k, c in enumerate(markers_list)}
    if max_len < 1:
        return oracle.E_NO_PATH, None
    segs = {}
    for k, c in enumerate(markers_list):
        segs[k] = _segment(m, c, markers, max_len, first_step_from=m[c[1], c[0]])
    if start in markers:  # the robot stands on a marker: walker 0 ends there at once
        st, cells, nxt = 3, [], markers[start]
    else:
        st, cells, nxt = _segment(m, start, markers, max_len)
    path = [start] + cells
    seen = set()
    while st == 3:
        if nxt in seen:
            return oracle.E_NO_PATH, None
        seen.add(nxt)
        st, c2, nxt2 = segs[nxt]
        path += c2
        nxt = nxt2
        if len(path) > max_len:
            return oracle.E_NO_PATH, None
    return (oracle.OK, np.array(path, np.int32)) if st == 1 else (oracle.E_NO_PATH, None)


def _fields(seed):
    static, goal, start = random_small_map(seed, N=40)
    cls = static.astype(np.uint8).copy()
    cls[goal[1], goal[0]] = oracle.GOAL
    out = []
    for sweeps in (0, 5, 60, 4000):
        u = oracle.init_u32(cls)
        oracle.relax_f32(cls, u, sweeps, max(sweeps, 1), 0.0)
        out.append((cls, u, (int(start[0]), int(start[1]))))
    return out


@pytest.mark.parametrize("seed", range(12))
def test_any_markers_give_the_single_walk(seed):
    rng = np.random.default_rng(seed)
    for cls, u, start in _fields(seed):
        m = oracle.index_matrix(cls, u)
        H, W = u.shape
        for max_len in (4 * (W + H), 30):
            ref_st, ref_cells = oracle.walk(cls, u, start, max_len)
            # markers: on the walk itself (when there is one), random cells, and the start cell
            for trial in range(6):
                cand = [tuple(map(int, c)) for c in rng.integers(0, [W, H], size=(rng.integers(0, 40), 2))]
                if ref_st == oracle.OK and len(ref_cells) > 2 and trial % 2 == 0:
                    idx = rng.choice(len(ref_cells), size=min(10, len(ref_cells)), replace=False)
                    cand += [tuple(map(int, ref_cells[i])) for i in idx]
                if trial == 5:
                    cand.append(start)
                markers = list(dict.fromkeys(cand))  # distinct, first occurrence kept
                st, cells = spec_walk(m, start, markers, max_len)
                assert st == ref_st, (seed, max_len, trial)
                if st == oracle.OK:
                    assert np.array_equal(cells, ref_cells), (seed, max_len, trial)
