"""Row-slab decomposition on the CPU: world_size 2 and 3 over torch.distributed
(gloo, 127.0.0.1), each rank relaxing its slab with the oracle; the gathered owned rows must be
bit-identical to the full-grid oracle relaxation, with the same sweeps and residual."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1903_07441_b200.slab import (SlabLayout, SlabRelaxer, DistExchanger, interval_schedule, slab_rows,
                                        sharded_walk, WALK_GOAL)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(W=70, H=61, seed=3):
    import oracle
    rng = np.random.default_rng(seed)
    cls = (rng.random((H, W)) < 0.1).astype(np.uint8)
    cls[H // 3, W // 2] = oracle.GOAL
    u = oracle.init_u32(cls)
    return cls, u


class OracleSlabBackend:
    """Test backend: the oracle relaxes the local grid (owned + ghosts, outside = obstacle)."""

    def __init__(self, lay, cls_g, u_g):
        import oracle
        self.o, self.lay = oracle, lay
        self.cls = np.ascontiguousarray(lay.local_slice(cls_g, 1))
        self.u = np.ascontiguousarray(lay.local_slice(u_g, np.float32(0)))
        self.t = torch.from_numpy(self.u)

    def relax(self, n, need_residual=True):
        lay = self.lay
        _, r = self.o.relax_f32_ex(self.cls, self.u, n, n, 0.0, row_parity=lay.row_offset,
                                   res_rows=(lay.G, lay.local_h - lay.G))
        return r

    def field_view(self):
        return self.t

    def walk_segment(self, x, yl, max_cells):
        """Follow the oracle's index matrix of the local grid inside the owned rows (test backend)."""
        m = self.o.index_matrix(self.cls, self.u)
        lay = self.lay
        cells = [(x, yl)]
        steps = ((1, 0), (-1, 0), (0, 1), (0, -1))
        if max_cells < 1:
            return -5, [], None
        while True:
            d = int(m[yl, x])
            if d == 4:
                return 0, cells, None
            if d >= 5:
                return -5, [], None
            nx, ny = x + steps[d][0], yl + steps[d][1]
            if ny < lay.G or ny >= lay.local_h - lay.G:
                return (1 if ny < lay.G else 2), cells, (nx, ny)
            if len(cells) + 1 > max_cells:
                return -5, [], None
            x, yl = nx, ny
            cells.append((x, yl))


def _walk_worker(rank, world, port, k, S, start, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cls, u = _problem()
    H, W = cls.shape
    lay = SlabLayout(W, H, world, rank, k)
    be = OracleSlabBackend(lay, cls, u)
    ex = DistExchanger()
    SlabRelaxer(be, lay, ex).relax(S)
    code, mine, total = sharded_walk(be, lay, ex, start, 4 * W * H)
    segs = [None] * world
    dist.all_gather_object(segs, [(c, np.asarray(sg).tolist()) for c, sg in mine])
    if rank == 0:
        parts = sorted([p for r in segs for p in r], key=lambda t: t[0])
        cells = [xy for _, sg in parts for xy in sg]
        out.put((code, total, cells))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k", [(2, 2), (3, 4)])
def test_sharded_walk_gloo_equals_single_grid(world, k):
    import oracle
    S = 3000
    start = (3, 58)  # bottom slab; the goal (35, 20) lies in the top one
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_walk_worker, args=(r, world, port, k, S, start, q)) for r in range(world)]
    for p in procs:
        p.start()
    code, total, cells = q.get(timeout=180)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    cls, u = _problem()
    oracle.relax_f32(cls, u, S, S, 0.0)
    st, ref = oracle.walk(cls, u, start, 4 * cls.size)
    assert st == oracle.OK and code == WALK_GOAL
    assert total == len(ref) and np.array_equal(np.asarray(cells), ref)
    rows = {slab_rows(cls.shape[0], world, r) for r in range(world)}
    assert len({next(i for i, (a, b) in enumerate(sorted(rows)) if a <= y < b) for _, y in ref}) > 1  # crosses slabs


def _worker(rank, world, port, k, S, check_every, tol, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cls, u = _problem()
    H, W = cls.shape
    lay = SlabLayout(W, H, world, rank, k)
    be = OracleSlabBackend(lay, cls, u)
    s, res = SlabRelaxer(be, lay, DistExchanger()).relax(S, check_every, tol)
    full = torch.zeros((H, W), dtype=torch.float32)  # owned rows in place, zeros elsewhere: a sum is exact
    full[lay.r0:lay.r1] = torch.from_numpy(be.u[lay.G:lay.local_h - lay.G].copy())
    dist.all_reduce(full, op=dist.ReduceOp.SUM)
    if rank == 0:
        out.put((s, res, full.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k,S,check_every,tol", [(2, 2, 37, 0, 0.0), (3, 4, 50, 0, 0.0), (2, 3, 4000, 6, 2e-4)])
def test_row_slabs_gloo_bit_identical(world, k, S, check_every, tol):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, S, check_every, tol, q)) for r in range(world)]
    for p in procs:
        p.start()
    s, res, field = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    cls, u = _problem()
    s_ref, r_ref = oracle.relax_f32(cls, u, S, check_every or S, tol)
    assert s == s_ref and np.float32(res) == np.float32(r_ref)
    assert np.array_equal(field, u)


def test_interval_schedule_respects_checks():
    sched = list(interval_schedule(23, 4, check_every=6, tol=1e-3))
    assert [n for n, _, _ in sched] == [4, 2, 4, 2, 4, 2, 4, 1]
    assert [s for _, c, s in sched if c] == [6, 12, 18, 23]
    assert [n for n, _, _ in interval_schedule(10, 4)] == [4, 4, 2]


def test_slab_layout():
    lay = SlabLayout(10, 100, 3, 1, 4)
    assert (lay.r0, lay.r1, lay.G, lay.local_h, lay.row_offset) == (34, 67, 8, 49, 26)
    assert sum(b - a for a, b in (slab_rows(100, 3, r) for r in range(3))) == 100
    with pytest.raises(ValueError):
        SlabLayout(10, 20, 4, 0, 4)
