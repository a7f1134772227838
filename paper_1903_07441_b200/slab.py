"""Row-slab decomposition of the relaxation across ranks (BASELINE.json configs[3]).

Each rank owns a contiguous block of global rows [r0, r1) and keeps G = 2k ghost rows above and
below it.  It relaxes its local grid (owned + ghosts) for k sweeps with ``twg_relax``; rows within
2k of the local edge are then stale, which is exactly the ghost region, so the owned rows are
bit-identical to a single-grid relaxation (the outermost ghost row is read-only and the inner
2k - 1 are recomputed redundantly; SURVEY.md §0 finding 6).  Then the 2k owned boundary rows are
sent to each neighbour and its ghost rows received (NCCL point-to-point through
``torch.distributed`` on GPUs, gloo on the CPU).  At check sweeps the owned-row residuals are
max-all-reduced, so every rank applies the same stop rule (C6).  Colours stay global because
each slab is created with ``row_offset = r0 - G`` (C1).

The compute backend is pluggable (``relax(n) -> residual``, ``field_view() -> [rows, pitch]``):
:class:`TwgSlabBackend` wraps a libtwg context; the CPU tests drive the same schedule with the
oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def slab_rows(H: int, world: int, rank: int):
    """Owned global rows [r0, r1) of `rank` (near-equal contiguous split)."""
    base, extra = divmod(H, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


@dataclass
class SlabLayout:
    W: int
    H_global: int
    world: int
    rank: int
    k: int  # sweeps between ghost exchanges

    def __post_init__(self):
        self.G = 2 * self.k
        self.r0, self.r1 = slab_rows(self.H_global, self.world, self.rank)
        if self.r1 - self.r0 < self.G:
            raise ValueError(f"slab of {self.r1 - self.r0} rows is thinner than 2k = {self.G}")
        self.local_h = self.r1 - self.r0 + 2 * self.G
        self.row_offset = self.r0 - self.G  # global index of local row 0

    # local row ranges
    def ghost_top(self):
        return 0, self.G

    def owned_top(self):
        return self.G, 2 * self.G

    def owned_bottom(self):
        return self.local_h - 2 * self.G, self.local_h - self.G

    def ghost_bottom(self):
        return self.local_h - self.G, self.local_h

    def global_rows(self):
        """Global rows covered by the local grid (ghost rows outside the grid are padding)."""
        return self.row_offset, self.row_offset + self.local_h

    def local_slice(self, global_array, fill):
        """Rows row_offset .. row_offset + local_h of a global [H, W] array; rows outside -> fill."""
        out = np.full((self.local_h,) + global_array.shape[1:], fill, dtype=global_array.dtype)
        g0, g1 = self.global_rows()
        a, b = max(g0, 0), min(g1, self.H_global)
        out[a - g0:b - g0] = global_array[a:b]
        return out


def interval_schedule(max_sweeps: int, k: int, check_every: int = 0, tol: float = 0.0):
    """Yield (n, is_check): n sweeps between exchanges, never crossing a check sweep."""
    ce = check_every if (tol > 0 and check_every > 0) else max(max_sweeps, 1)
    s = 0
    while s < max_sweeps:
        nxt = (s // ce + 1) * ce
        n = min(k, nxt - s, max_sweeps - s)
        s += n
        yield n, (s % ce == 0) or s == max_sweeps, s


class DistExchanger:
    """Ghost exchange and residual reduction over torch.distributed (NCCL or gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def exchange(self, lay: SlabLayout, field):
        d = self.dist
        ops = []
        if lay.rank > 0:
            a, b = lay.owned_top()
            ops.append(d.P2POp(d.isend, field[a:b].contiguous(), lay.rank - 1, self.group))
            ga, gb = lay.ghost_top()
            top = field[ga:gb]
            rt = top if top.is_contiguous() else top.contiguous()
            ops.append(d.P2POp(d.irecv, rt, lay.rank - 1, self.group))
        if lay.rank < lay.world - 1:
            a, b = lay.owned_bottom()
            ops.append(d.P2POp(d.isend, field[a:b].contiguous(), lay.rank + 1, self.group))
            ga, gb = lay.ghost_bottom()
            bot = field[ga:gb]
            rb = bot if bot.is_contiguous() else bot.contiguous()
            ops.append(d.P2POp(d.irecv, rb, lay.rank + 1, self.group))
        if ops:
            for r in d.batch_isend_irecv(ops):
                r.wait()

    def broadcast_from(self, owner: int, values, device=None):
        """Small int64 message from rank `owner` to every rank (a SUM all-reduce of zeros elsewhere)."""
        import torch
        t = torch.tensor(values if self.dist.get_rank() == owner else [0] * len(values), dtype=torch.int64,
                         device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return [int(v) for v in t.tolist()]

    def allreduce_max(self, value: float, device=None) -> float:
        import torch
        t = torch.tensor([value], dtype=torch.float32, device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


class SlabRelaxer:
    """Runs the k-sweep interval schedule of one rank."""

    def __init__(self, backend, layout: SlabLayout, exchanger, device=None):
        self.backend, self.lay, self.ex, self.device = backend, layout, exchanger, device

    def relax(self, max_sweeps: int, check_every: int = 0, tol: float = 0.0):
        res, s = 0.0, 0
        for n, is_check, s in interval_schedule(max_sweeps, self.lay.k, check_every, tol):
            r = self.backend.relax(n, need_residual=is_check)
            if is_check:
                res = self.ex.allreduce_max(r, self.device)
            if s < max_sweeps:
                self.ex.exchange(self.lay, self.backend.field_view())
            if is_check and tol > 0 and check_every > 0 and s % check_every == 0 and res < tol:
                break
        return s, res


class _CudaView:
    """Zero-copy torch view of a device buffer (``__cuda_array_interface__``)."""

    def __init__(self, ptr, shape, typestr="<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class TwgSlabBackend:
    """libtwg context holding one slab: local grid = owned rows + 2G ghost rows."""

    def __init__(self, planner, device=0):
        self.pl = planner
        self.device = device

    def relax(self, n: int, need_residual: bool = True) -> float:
        """n sweeps; the residual is read back (a host synchronisation) only when asked for."""
        from .twg import relax_cfg
        _, res = self.pl.relax(relax_cfg(max_sweeps=n), want_result=need_residual)
        return float(res[0]) if need_residual else 0.0

    def walk_segment(self, x: int, yl: int, max_cells: int):
        """Walk from local cell (x, yl) until the goal, a hand-over or a dead end (twg_walk_from)."""
        return self.pl.walk_from(0, x, yl, max_cells)

    def field_view(self):
        import torch
        ptr, pitch = self.pl.field_ptr(0)
        return torch.as_tensor(_CudaView(ptr, (self.pl.H, pitch)), device=f"cuda:{self.device}")


def make_twg_slab(layout: SlabLayout, static_global, robot, goal, tracks, warp, cell_size=0.1,
                  origin=(0.0, 0.0), device=0, stream=None):
    """Create and encode (cold) the libtwg context of one slab from the global scene.

    Local row 0 is global row ``layout.row_offset``; ghost rows outside the global grid are walls
    (outside = obstacle, C4).  The goal is passed in local coordinates (it may lie outside)."""
    from .twg import Planner
    pl = Planner(layout.W, layout.local_h, 1, cell_size, (origin[0], origin[1] + layout.row_offset * cell_size),
                 device=device, stream=stream, row_offset=layout.row_offset, ghost_rows=layout.G)
    pl.set_static(np.ascontiguousarray(layout.local_slice(np.asarray(static_global, np.uint8), 1)))
    pl.set_obstacles(0, robot, (goal[0], goal[1] - layout.row_offset), tracks, warp, warm=0)
    return pl


def nccl_comm_for(rank: int, world: int, device: int, group=None) -> int:
    """An NCCL communicator for the libtwg sharded contexts (twg_nccl_comm_init): rank 0 draws the
    unique id (twg_nccl_unique_id) and torch.distributed broadcasts it (any backend)."""
    import torch.distributed as dist
    from .twg import nccl_comm_init, nccl_unique_id
    obj = [nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0, group=group)
    return nccl_comm_init(world, obj[0], rank, device)


def make_sharded(W, H, static_global, robot, goal, tracks, warp, k, nccl_comm, cell_size=0.1, origin=(0.0, 0.0),
                 device=0, stream=None):
    """This rank's slab of the global grid as a libtwg sharded context (twg_create with nccl_comm): the
    library exchanges the ghost rows and reduces the residual inside twg_relax.  Encoded cold."""
    from .twg import Planner
    pl = Planner(W, H, 1, cell_size, origin, device=device, stream=stream, nccl_comm=nccl_comm, exchange_every=k)
    pl.set_static(np.ascontiguousarray(np.asarray(static_global, np.uint8)))
    pl.set_obstacles(0, robot, goal, tracks, warp, warm=0)
    return pl


def make_group(W, H, nslabs, static_global, robot, goal, tracks, warp, k, cell_size=0.1, origin=(0.0, 0.0),
               device=0, stream=None):
    """nslabs slabs of one global grid on one device (twg_create_group), encoded cold."""
    from .twg import Planner
    pls = Planner.create_group(W, H, nslabs, k, cell_size, origin, device, stream)
    for pl in pls:
        pl.set_static(np.ascontiguousarray(np.asarray(static_global, np.uint8)))
        pl.set_obstacles(0, robot, goal, tracks, warp, warm=0)
    return pls


def owned_rows(pl, mode=0):
    """The owned rows [r0, r1) of a slab context's field (twg_get_field returns the local slab)."""
    f = pl.get_field(0, mode)
    return f[pl.ghost_rows:pl.H - pl.ghost_rows]


def exchange_local(backends, layouts):
    """Ghost-row exchange between slabs held by one process (device-to-device copies)."""
    views = [b.field_view() for b in backends]
    for r in range(len(backends) - 1):
        up, dn, lu, ld = views[r], views[r + 1], layouts[r], layouts[r + 1]
        a, b = lu.owned_bottom()
        ga, gb = ld.ghost_top()
        top_src = up[a:b].clone()
        a2, b2 = ld.owned_top()
        ga2, gb2 = lu.ghost_bottom()
        bot_src = dn[a2:b2].clone()
        dn[ga:gb].copy_(top_src)
        up[ga2:gb2].copy_(bot_src)


def relax_local_slabs(backends, layouts, max_sweeps: int, check_every: int = 0, tol: float = 0.0):
    """All slabs in one process (e.g. several contexts on one GPU): the same interval schedule,
    ghost rows copied between the slabs' buffers, residual = max over slabs."""
    k = layouts[0].k
    res, s = 0.0, 0
    for n, is_check, s in interval_schedule(max_sweeps, k, check_every, tol):
        rs = [b.relax(n, need_residual=is_check) for b in backends]
        if is_check:
            res = max(rs)
        if s < max_sweeps:
            exchange_local(backends, layouts)
        if is_check and tol > 0 and check_every > 0 and s % check_every == 0 and res < tol:
            break
    return s, res


WALK_GOAL, WALK_UP, WALK_DOWN, WALK_NO_PATH = 0, 1, 2, -5


def owner_of_row(H: int, world: int, gy: int) -> int:
    for r in range(world):
        r0, r1 = slab_rows(H, world, r)
        if r0 <= gy < r1:
            return r
    raise ValueError(f"row {gy} outside the grid")


def sharded_walk(backend, lay: SlabLayout, ex, start, max_len: int, device=None):
    """Descent walk over row slabs: the rank owning the current cell walks until the
    goal, a dead end, or the first step into another slab, then hands the walker (next cell and cells
    so far) to that neighbour with one small message.  Ghost rows are exchanged first so every rank
    sees its neighbours' final rows.  Returns (code, this rank's cells in global coordinates, total
    cell count); concatenating the ranks' cells in walk order gives the single-grid walk."""
    ex.exchange(lay, backend.field_view())
    x, gy = int(start[0]), int(start[1])
    owner = owner_of_row(lay.H_global, lay.world, gy)
    count = 0
    mine = []
    while True:
        if lay.rank == owner:
            code, seg, nxt = backend.walk_segment(x, gy - lay.row_offset, max_len - count)
            if code != WALK_NO_PATH and len(seg):
                seg = np.asarray(seg).copy()
                seg[:, 1] += lay.row_offset
                mine.append((count, seg))
            n = len(seg) if code != WALK_NO_PATH else 0
            msg = [code, nxt[0] if nxt else -1, (nxt[1] + lay.row_offset) if nxt else -1, count + n]
        else:
            msg = [0, 0, 0, 0]
        code, nx, ny, count = ex.broadcast_from(owner, msg, device)
        if code == WALK_NO_PATH:
            return code, [], 0
        if code == WALK_GOAL:
            return code, mine, count
        owner += -1 if code == WALK_UP else 1
        x, gy = nx, ny


def sharded_walk_local(backends, layouts, start, max_len: int):
    """The same hand-over on several slabs held by one process (ghost rows already exchanged)."""
    lay0 = layouts[0]
    x, gy = int(start[0]), int(start[1])
    owner = owner_of_row(lay0.H_global, lay0.world, gy)
    cells = []
    while True:
        lay = layouts[owner]
        code, seg, nxt = backends[owner].walk_segment(x, gy - lay.row_offset, max_len - len(cells))
        if code == WALK_NO_PATH:
            return code, np.zeros((0, 2), np.int32)
        seg = np.asarray(seg).copy()
        seg[:, 1] += lay.row_offset
        cells.extend(seg.tolist())
        if code == WALK_GOAL:
            return code, np.asarray(cells, np.int32)
        owner += -1 if code == WALK_UP else 1
        x, gy = nxt[0], nxt[1] + lay.row_offset
