"""Multi-rank path on CPU (gloo, world sizes 2 and 3): the H3D wz partition, the
static tile halo plan and the exchange orchestration of paper_2208_11617_b200.dist,
with the CPU oracle standing in for the per-rank step (test infrastructure only).

Non-owned cells are poisoned after every local step, so the result is correct
only if every tile a rank reads arrives through the halo plan."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import BB, H3D, Restated, tet_cells
from paper_2208_11617_b200 import dist as D


def tile_cells(side, rho, tiles):
    """(k, rho^3) packed indices (or -1) of every tile's cells, lz, ly, lx order."""
    l = np.arange(rho)
    lz, ly, lx = np.meshgrid(l, l, l, indexing="ij")
    t = np.asarray(tiles, np.int64).reshape(-1, 3)
    cx = t[:, 0, None] * rho + lx.ravel()[None]
    cy = t[:, 1, None] * rho + ly.ravel()[None]
    cz = t[:, 2, None] * rho + lz.ravel()[None]
    ok = D.tet_contains(side, cx, cy, cz)
    idx = np.where(ok, D.tet_index(side, np.where(ok, cx, 0), np.where(ok, cy, 0), np.where(ok, cz, 0)), -1)
    return idx


class OracleOps:
    """CPU stand-in for CudaOps: oracle full step, keep own tiles, poison the rest."""

    def __init__(self, orc, side, rho, own_idx, seed):
        self.orc, self.side, self.rho = orc, side, rho
        self.own = np.zeros(tet_cells(side), bool)
        self.own[own_idx[own_idx >= 0]] = True
        self.rng = np.random.default_rng(seed)

    def step_range(self, cur, nxt, lo, hi):
        c = cur.numpy().copy()
        self.orc.ca3d_run(self.side, 1, c, threads=1)
        n = nxt.numpy()
        n[:] = self.rng.integers(0, 2, n.size, dtype=np.uint8)
        n[self.own] = c[self.own]

    def pack(self, cells, tiles, out):
        idx = tile_cells(self.side, self.rho, tiles.numpy())
        v = np.where(idx >= 0, cells.numpy()[np.maximum(idx, 0)], 0).astype(np.uint8)
        out.numpy()[:] = v.ravel()

    def unpack(self, cells, tiles, buf):
        idx = tile_cells(self.side, self.rho, tiles.numpy()).ravel()
        b = buf.numpy()
        m = idx >= 0
        cells.numpy()[idx[m]] = b[m]

    def empty(self, n):
        return torch.zeros(max(n, 1), dtype=torch.uint8)

    def tiles(self, t):
        return torch.from_numpy(np.ascontiguousarray(t, dtype=np.int32).reshape(-1, 3))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, n, rho, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Restated()
    m = 3
    outcomes = orc.map_outcomes(kind, m, n)
    ext = orc.grid(kind, m, n)
    strict = kind == H3D
    dom_blocks = n - 1 if strict else n
    side = dom_blocks * rho
    plan = D.build_plan(ext, outcomes, strict, dom_blocks, world)
    own_idx = tile_cells(side, rho, plan.owned_tiles[rank])
    ops = OracleOps(orc, side, rho, own_idx, seed=rank + 7)
    sh = D.ShardedLife(plan, rank, rho, ops)
    cur = torch.from_numpy(orc.make_life_state(3, side, 42, threads=1))
    nxt = torch.zeros_like(cur)
    res = sh.run(cur, nxt, steps)
    sh.gather_owned(res, 0)
    if rank == 0:
        want = orc.make_life_state(3, side, 42, threads=1)
        orc.ca3d_run(side, steps, want, threads=1)
        q.put((bool((res.numpy() == want).all()), plan.wz_ranges, [plan.halo_tiles(r) for r in range(world)]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,n,rho,steps", [(2, H3D, 16, 2, 4), (3, H3D, 16, 2, 3), (2, BB, 15, 2, 3),
                                                    (2, H3D, 32, 1, 3)])
def test_sharded_life_matches_oracle(world, kind, n, rho, steps):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, n, rho, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok, ranges, halos = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok, (ranges, halos)
    assert len(ranges) == world and ranges[0][0] == 0
    assert all(h > 0 for h in halos)


def test_partition_balanced_whole_levels():
    orc = Restated()
    for n, world in [(64, 8), (128, 8), (32, 2)]:
        out = orc.map_outcomes(H3D, 3, n)
        ext = orc.grid(H3D, 3, n)
        plan = D.build_plan(ext, out, True, n - 1, world)
        counts = [t.shape[0] for t in plan.owned_tiles]
        assert sum(counts) == tet_cells(n - 1)
        assert max(counts) / (sum(counts) / world) < 1.15
        # contiguous, covering wz ranges
        assert plan.wz_ranges[0][0] == 0 and plan.wz_ranges[-1][1] == ext[2]
        assert all(a[1] == b[0] for a, b in zip(plan.wz_ranges, plan.wz_ranges[1:]))
        # halo symmetric bookkeeping: what q sends r is what r receives from q
        for r in range(world):
            for q, t in plan.recv(r).items():
                assert (plan.send[q][r] == t).all()


def test_partition_rows_balanced_and_contiguous():
    """ACCUM / MAP row sharding: contiguous row ranges covering
    the grid, balanced by useful blocks within one row's weight."""
    from oracle.oracle import BB, H2D, Restated
    from paper_2208_11617_b200 import dist as D
    o = Restated()
    for kind, n, ex, ey in ((H2D, 64, 32, 63), (BB, 63, 63, 63), (H2D, 1024, 512, 1023)):
        u = D.useful_per_row(o.map_outcomes(kind, 2, n), ex, ey)
        for world in (1, 2, 3, 8):
            r = D.partition_rows(u, world)
            assert r[0][0] == 0 and r[-1][1] == ey
            assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))
            loads = [int(u[lo:hi].sum()) for lo, hi in r]
            assert max(loads) - int(u.sum()) / world <= int(u.max()), (kind, n, world, loads)


class EngineCpuOps:
    """CPU stand-in for EngineOps (ShardedEngine): chunks are tiles (merged in
    x-adjacent pairs, so multi-tile chunks are exercised), run_list writes the
    oracle's next state on the chunk's tiles only, every other cell of the
    output is poisoned at the start of a step, halo tiles travel as u8 tiles."""

    def __init__(self, orc, kind, n, rho, side, seed):
        self.orc, self.kind, self.n, self.rho, self.side = orc, kind, n, rho, side
        self.rng = np.random.default_rng(seed)
        self.tile_bytes = rho ** 3
        self._next = None
        base = OracleOps(orc, side, rho, np.zeros(0, np.int64), seed)
        self.pack, self.unpack, self.empty, self.tiles = base.pack, base.unpack, base.empty, base.tiles

    def plan(self, lo, hi):
        o = self.orc.map_outcomes(self.kind, 3, self.n)
        ex, ey, _ = self.orc.grid(self.kind, 3, self.n)
        wz = np.arange(o.shape[0]) // (ex * ey)
        sel = (o[:, 0] == 0) & (wz >= lo) & (wz < hi)
        t = o[sel][:, 1:4].astype(np.int64)
        if self.kind == H3D:
            t[:, 1] -= 1
        t = t[np.lexsort((t[:, 0], t[:, 1], t[:, 2]))]
        out, i = [], 0
        while i < t.shape[0]:
            j = i + 1
            if j < t.shape[0] and (t[j, 1:] == t[i, 1:]).all() and t[j, 0] == t[i, 0] + 1:
                j += 1
            r = self.rho
            out.append((t[i, 0] * r, t[i, 1] * r, t[i, 2] * r, (j - i) * r))
            i = j
        return np.asarray(out, np.int32).reshape(-1, 4)

    def chunks(self, arr):
        return arr

    def begin_step(self, b):
        self._next = None
        b.numpy()[:] = self.rng.integers(0, 2, b.numel(), dtype=np.uint8)

    def run_list(self, a, b, chunks):
        if self._next is None:
            c = a.numpy().copy()
            self.orc.ca3d_run(self.side, 1, c, threads=1)
            self._next = c
        tx0, ty, tz, nt = D.chunk_tiles(chunks, self.rho)
        tl = [(x, y, z) for x0, y, z, k in zip(tx0, ty, tz, nt) for x in range(x0, x0 + k)]
        if tl:
            idx = tile_cells(self.side, self.rho, np.asarray(tl)).ravel()
            idx = idx[idx >= 0]
            b.numpy()[idx] = self._next[idx]

    def fork(self):
        import contextlib
        return contextlib.nullcontext()

    def join(self):
        pass


def _engine_worker(rank, world, port, kind, n, rho, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Restated()
    outcomes = orc.map_outcomes(kind, 3, n)
    ext = orc.grid(kind, 3, n)
    strict = kind == H3D
    dom_blocks = n - 1 if strict else n
    side = dom_blocks * rho
    plan = D.build_plan(ext, outcomes, strict, dom_blocks, world)
    ops = EngineCpuOps(orc, kind, n, rho, side, seed=rank + 11)
    eng = D.ShardedEngine(plan, rank, rho, ops)
    a = torch.from_numpy(orc.make_life_state(3, side, 42, threads=1))
    b = torch.zeros_like(a)
    res = eng.run(a, b, steps)
    sh = D.ShardedLife(plan, rank, rho, OracleOps(orc, side, rho, np.zeros(0, np.int64), 0))
    sh.gather_owned(res, 0)
    if rank == 0:
        want = orc.make_life_state(3, side, 42, threads=1)
        orc.ca3d_run(side, steps, want, threads=1)
        q.put((bool((res.numpy() == want).all()), eng.n_boundary, eng.n_interior))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,world", [(H3D, 16, 2), (H3D, 16, 3), (BB, 15, 2)])
def test_sharded_engine_schedule(kind, n, world):
    """The sharded engine's schedule (boundary chunks, pack + exchange, interior,
    unpack) with poisoned non-owned cells: exact after 3 steps only if the
    boundary/interior split and the halo plan are right."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_engine_worker, args=(r, world, port, kind, n, 4, 3, q)) for r in range(world)]
    for p in ps:
        p.start()
    ok, nb, ni = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
    assert nb > 0 and ni > 0


def test_split_chunks():
    # chunks of 2 tiles at rho = 4; tile (5, 7, 1) is sent -> only chunk 0
    ch = np.array([[16, 28, 4, 8], [40, 28, 4, 8], [0, 0, 0, 4]], np.int32)
    b, i = D.split_chunks(ch, np.array([[5, 7, 1]]), 16, 4)
    assert b.tolist() == [[16, 28, 4, 8]] and i.shape == (2, 4)
    b, i = D.split_chunks(ch, np.zeros((0, 3)), 16, 4)
    assert b.shape == (0, 4) and i.shape == (3, 4)
