"""f3 per-cell rubber band on the index matrix (Alg. 1, reading C37): twg_band_index's
optimised matrix and the walk along it bit-exact against orc_cellband / orc_walk_dir on the same
fields (the oracle's relaxation, bit-identical to libtwg's)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, warp_cfg  # noqa: E402
from paper_1903_07441_b200 import twg as T  # noqa: E402
from scenes import scene_c1, scene_random  # noqa: E402


def _run(sc, sweeps, iters, kt, max_len=20000):
    st = torch.cuda.current_stream().cuda_stream
    pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, st)
    pl.set_static(sc.static)
    pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
    pl.relax(relax_cfg(max_sweeps=sweeps))
    s, m, cells = pl.band_index(0, band_cfg(iters, max_len, 8, k_t=kt))
    ost, cls, *_ = oracle.classify(sc)
    u = oracle.init_u32(cls)
    oracle.relax_f32(cls, u, sweeps, sweeps, 0.0)
    assert np.array_equal(pl.get_field(0, 1), u)
    ref = oracle.cellband(cls, u, oracle.index_matrix(cls, u), iters, kt)
    assert np.array_equal(m, ref)
    wst, wref = oracle.walk_dir(ref, oracle.robot_cell(sc), max_len)
    assert (s == T.OK) == (wst == oracle.OK)
    assert np.array_equal(cells, wref)
    pl.close()
    return s, m, ref


@pytest.mark.parametrize("iters,kt", [(0, 1.0), (1, 1.0), (5, 0.5), (50, 1.0), (20, 2.0)])
def test_cellband_c1(iters, kt):
    _run(scene_c1(), 3000, iters, kt)


@pytest.mark.parametrize("seed", [3, 8])
def test_cellband_random_scenes(seed):
    _run(scene_random("cb", 150, 4, 8, seed), 20000, 30, 1.0)


def test_cellband_ragged_width():
    _run(scene_random("cbr", 77, 2, 3, 5), 8000, 10, 1.0)
