"""Row slabs inside libtwg: sharded contexts whose twg_relax runs the
exchange intervals itself -- shrinking ghost ranges, the boundary/interior split of the last launch
of an interval on two streams, the ghost exchange (device copies for a local group, ncclSend /
ncclRecv for an NCCL communicator) and the on-device residual max before the stop rule.  The owned
rows must be bit-identical to one full-grid context and to the oracle (Eq. 2)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg  # noqa: E402
from paper_1903_07441_b200 import twg as T  # noqa: E402
from paper_1903_07441_b200.slab import (SlabLayout, TwgSlabBackend, make_group, make_sharded, nccl_comm_for,  # noqa: E402
                                        owned_rows, sharded_walk_local, WALK_GOAL)
from paper_1903_07441_b200.twg import nccl_comm_destroy  # noqa: E402
from scenes import scene_random  # noqa: E402


def _full(sc, S, check_every, tol, T=0):
    st = torch.cuda.current_stream().cuda_stream
    full = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, st)
    full.set_static(sc.static)
    full.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    sw, rs = full.relax(relax_cfg(max_sweeps=S, check_every=check_every, tol=tol, temporal_depth=T))
    ref = full.get_field(0, 0)
    full.close()
    return int(sw[0]), float(rs[0]), ref


@pytest.mark.parametrize("nslabs,k,S,check_every,tol,T", [
    (2, 12, 96, 0, 0.0, 0),      # two T = 6 launches per interval (shrinking ghosts), split last launch
    (3, 5, 101, 0, 0.0, 0),      # k < T: one 5-sweep launch per interval, remainder interval
    (4, 13, 77, 0, 0.0, 4),      # T = 4: launches 4, 4, 4, 1
    (2, 8, 3000, 8, 5e-4, 0),    # tolerance stop: the residual max is reduced across the slabs
    (5, 3, 40, 0, 0.0, 2),       # launches 2 + 1 per interval
    (10, 6, 61, 0, 0.0, 0),      # thin slabs (30 rows, G = 12): no split; one launch per interval, so
                                 # the field alternates buffers between intervals
])
def test_group_slabs_bit_identical(nslabs, k, S, check_every, tol, T):
    sc = scene_random("gslab", 300, 12, 25, 5)
    sw, rs, ref = _full(sc, S, check_every, tol, T)
    st = torch.cuda.current_stream().cuda_stream
    pls = make_group(sc.W, sc.H, nslabs, sc.static, sc.robot, sc.goal, sc.tracks, warp_cfg(), k, stream=st)
    s, res = pls[0].relax(relax_cfg(max_sweeps=S, check_every=check_every, tol=tol, temporal_depth=T))
    assert int(s[0]) == sw and np.float32(res[0]) == np.float32(rs)
    got = np.concatenate([owned_rows(p) for p in pls])
    assert got.shape == ref.shape
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    # the ghost rows hold the neighbours' final rows after the call
    for a, b in zip(pls[:-1], pls[1:]):
        fa, fb = a.get_field(0, 0), b.get_field(0, 0)
        G = a.ghost_rows
        assert np.array_equal(fa[a.H - G:].view(np.uint32), fb[G:2 * G].view(np.uint32))
        assert np.array_equal(fb[:G].view(np.uint32), fa[a.H - 2 * G:a.H - G].view(np.uint32))
    ost, cls, *_ = oracle.classify(sc)
    u = oracle.init_u32(cls)
    s_o, r_o = oracle.relax_f32(cls, u, S, check_every or S, tol)
    assert s_o == sw and np.float32(r_o) == np.float32(res[0])
    assert np.array_equal(np.abs(got), u)
    for p in pls:
        p.close()


def test_group_walk_hand_over():
    # the library-sharded group, then the walker handed from slab to slab == the oracle walk
    sc = scene_random("gslabw", 150, 4, 6, 8)
    st = torch.cuda.current_stream().cuda_stream
    nslabs, k, S = 3, 6, 20000
    pls = make_group(sc.W, sc.H, nslabs, sc.static, sc.robot, sc.goal, sc.tracks, warp_cfg(), k, stream=st)
    pls[0].relax(relax_cfg(max_sweeps=S))
    lays = [SlabLayout(sc.W, sc.H, nslabs, r, k) for r in range(nslabs)]
    assert [(p.r0, p.r1, p.row_offset) for p in pls] == [(l.r0, l.r1, l.row_offset) for l in lays]
    bes = [TwgSlabBackend(p) for p in pls]
    ost, cls, *_ = oracle.classify(sc)
    u = oracle.init_u32(cls)
    oracle.relax_f32(cls, u, S, S, 0.0)
    start = oracle.robot_cell(sc)
    wst, ref = oracle.walk(cls, u, start, 4 * sc.W * sc.H)
    code, cells = sharded_walk_local(bes, lays, start, 4 * sc.W * sc.H)  # ghosts already exchanged by twg_relax
    assert wst == oracle.OK and code == WALK_GOAL and np.array_equal(cells, ref)
    for p in pls:
        p.close()


@pytest.mark.parametrize("k,S,check_every,tol", [(12, 120, 0, 0.0), (7, 2000, 16, 1e-4)])
def test_nccl_slab_world_size_1(k, S, check_every, tol):
    # the NCCL path of twg_create / twg_relax (communicator of one rank: all-reduce, no neighbours)
    sc = scene_random("nslab", 256, 10, 20, 6)
    sw, rs, ref = _full(sc, S, check_every, tol)
    comm = nccl_comm_for(0, 1, 0)
    st = torch.cuda.current_stream().cuda_stream
    pl = make_sharded(sc.W, sc.H, sc.static, sc.robot, sc.goal, sc.tracks, warp_cfg(), k, comm, stream=st)
    assert (pl.rank, pl.nranks, pl.r0, pl.r1, pl.ghost_rows) == (0, 1, 0, sc.H, 2 * k)
    s, res = pl.relax(relax_cfg(max_sweeps=S, check_every=check_every, tol=tol))
    assert int(s[0]) == sw and np.float32(res[0]) == np.float32(rs)
    assert np.array_equal(owned_rows(pl).view(np.uint32), ref.view(np.uint32))
    pl.close()
    nccl_comm_destroy(comm)


@pytest.mark.parametrize("nslabs,k,iters", [(3, 6, 50), (4, 4, 20)])
def test_group_extract_path_equals_single_grid(nslabs, k, iters):
    # twg_extract_path on a local slab group: walk handed over between the slabs, band + resampling on
    # the gathered corridor -- cells, smoothed path and next waypoint bit-identical to the oracle's
    # single-grid plan step (every slab returns the same global path)
    sc = scene_random("gpath", 150, 4, 6, 8)
    st = torch.cuda.current_stream().cuda_stream
    S = 20000
    pls = make_group(sc.W, sc.H, nslabs, sc.static, sc.robot, sc.goal, sc.tracks, warp_cfg(), k, stream=st)
    pls[0].relax(relax_cfg(max_sweeps=S))
    ref = oracle.plan_step(sc, max_sweeps=S, iters=iters, max_len=4000)
    assert ref["walk_status"] == oracle.OK
    owners = {next(r for r, p in enumerate(pls) if p.r0 <= y < p.r1) for _, y in ref["cells"]}
    assert len(owners) > 1  # the walk crosses slabs
    for p in (pls[0], pls[-1]):
        s, cells, sm, ns, nxt = p.extract_path(0, band_cfg(iters, 4000, 8000))
        assert s == T.OK
        assert np.array_equal(cells, ref["cells"])
        assert np.array_equal(sm.view(np.uint32), ref["smooth"].view(np.uint32))
        assert nxt == ref["next"]
    for p in pls:
        p.close()


def test_nccl_slab_extract_path_world_size_1():
    sc = scene_random("npath", 128, 3, 6, 8)
    S = 20000
    comm = nccl_comm_for(0, 1, 0)
    st = torch.cuda.current_stream().cuda_stream
    pl = make_sharded(sc.W, sc.H, sc.static, sc.robot, sc.goal, sc.tracks, warp_cfg(), 6, comm, stream=st)
    pl.relax(relax_cfg(max_sweeps=S))
    ref = oracle.plan_step(sc, max_sweeps=S, iters=50, max_len=4000)
    s, cells, sm, ns, nxt = pl.extract_path(0, band_cfg(50, 4000, 8000))
    assert (s == T.OK) == (ref["walk_status"] == oracle.OK)
    if s == T.OK:
        assert np.array_equal(cells, ref["cells"])
        assert np.array_equal(sm.view(np.uint32), ref["smooth"].view(np.uint32)) and nxt == ref["next"]
    pl.close()
    nccl_comm_destroy(comm)
