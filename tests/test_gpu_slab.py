"""Row slabs on one GPU ("virtual slabs"): G libtwg contexts with ghost rows, the
same interval schedule as the multi-GPU path, ghosts copied between the contexts' buffers.  The
owned rows must be bit-identical to one full-grid context and to the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_1903_07441_b200 import Planner, relax_cfg, warp_cfg  # noqa: E402
from paper_1903_07441_b200.slab import (SlabLayout, TwgSlabBackend, make_twg_slab, relax_local_slabs,  # noqa: E402
                                        exchange_local, sharded_walk_local, WALK_GOAL)
from scenes import scene_random  # noqa: E402


@pytest.mark.parametrize("world,k,S,check_every,tol", [(2, 4, 64, 0, 0.0), (3, 8, 101, 0, 0.0), (4, 2, 37, 0, 0.0),
                                                      (2, 4, 3000, 8, 5e-4)])
def test_virtual_slabs_bit_identical(world, k, S, check_every, tol):
    sc = scene_random("slab", 300, 12, 25, 5)
    st = torch.cuda.current_stream().cuda_stream
    full = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, st)
    full.set_static(sc.static)
    full.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    sw, rs = full.relax(relax_cfg(max_sweeps=S, check_every=check_every, tol=tol))
    ref = full.get_field(0, 0)
    lays = [SlabLayout(sc.W, sc.H, world, r, k) for r in range(world)]
    pls = [make_twg_slab(l, sc.static, sc.robot, sc.goal, sc.tracks, warp_cfg(), stream=st) for l in lays]
    bes = [TwgSlabBackend(p) for p in pls]
    s, res = relax_local_slabs(bes, lays, S, check_every, tol)
    assert s == int(sw[0]) and np.float32(res) == np.float32(rs[0])
    got = np.concatenate([p.get_field(0, 0)[l.G:l.local_h - l.G] for p, l in zip(pls, lays)])
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    # and the oracle
    ost, cls, *_ = oracle.classify(sc)
    u = oracle.init_u32(cls)
    s_o, r_o = oracle.relax_f32(cls, u, S, check_every or S, tol)
    assert s_o == s and np.float32(r_o) == np.float32(res)
    assert np.array_equal(np.abs(got), u)


@pytest.mark.parametrize("world,k", [(2, 4), (4, 6)])
def test_virtual_slabs_sharded_walk(world, k):
    # walk handed from slab to slab (twg_walk_from) == the single-grid oracle walk
    sc = scene_random("slabw", 150, 4, 6, 8)
    st = torch.cuda.current_stream().cuda_stream
    S = 20000
    lays = [SlabLayout(sc.W, sc.H, world, r, k) for r in range(world)]
    pls = [make_twg_slab(l, sc.static, sc.robot, sc.goal, sc.tracks, warp_cfg(), stream=st) for l in lays]
    bes = [TwgSlabBackend(p) for p in pls]
    relax_local_slabs(bes, lays, S)
    exchange_local(bes, lays)
    ost, cls, *_ = oracle.classify(sc)
    u = oracle.init_u32(cls)
    oracle.relax_f32(cls, u, S, S, 0.0)
    start = oracle.robot_cell(sc)
    wst, ref = oracle.walk(cls, u, start, 4 * sc.W * sc.H)
    code, cells = sharded_walk_local(bes, lays, start, 4 * sc.W * sc.H)
    assert wst == oracle.OK and code == WALK_GOAL
    assert np.array_equal(cells, ref)
    owners = {next(r for r, l in enumerate(lays) if l.r0 <= y < l.r1) for _, y in ref}
    assert len(owners) > 1


def test_walk_from_unsharded_matches_extract_path():
    sc = scene_random("wf", 150, 4, 6, 4)
    st = torch.cuda.current_stream().cuda_stream
    pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, st)
    pl.set_static(sc.static)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    pl.relax(relax_cfg(max_sweeps=20000))
    from paper_1903_07441_b200 import band_cfg
    s, cells, *_ = pl.extract_path(0, band_cfg(0, 4000, 8000))
    rc = oracle.robot_cell(sc)
    code, c2, nxt = pl.walk_from(0, rc[0], rc[1], 4000)
    assert s == 0 and code == 0 and nxt is None and np.array_equal(c2, cells)
    code, c3, _ = pl.walk_from(0, rc[0], rc[1], 5)        # budget
    assert code == -5 and len(c3) == 0
