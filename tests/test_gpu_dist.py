"""The sharded 3-D Life path on ONE GPU: two ranks on cuda:0 run the real
sm_100a step-range and tile pack/unpack kernels; their halo travels over gloo
through host staging (NCCL rejects two ranks on one device). The orchestration
is paper_2208_11617_b200.dist.ShardedLife, unchanged."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, n, rho, ex, steps, q, bits=False, engine=False):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.oracle import Restated
    from paper_2208_11617_b200 import api
    from paper_2208_11617_b200 import dist as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    class StagedOps(D.CudaOps):
        def empty(self, n_):
            return torch.zeros(max(n_, 1), dtype=torch.uint8)  # host buffers for gloo

        def pack(self, cells, tiles, out):
            tmp = torch.empty(out.numel(), dtype=torch.uint8, device="cuda")
            super().pack(cells, tiles, tmp)
            out.copy_(tmp.cpu())

        def unpack(self, cells, tiles, buf):
            super().unpack(cells, tiles, buf.cuda())

    class StagedBitsOps(D.BitsOps):
        def empty(self, n_):
            return torch.zeros(max(n_, 1), dtype=torch.uint8)

        def pack(self, bits_, tiles, out):
            tmp = torch.empty(out.numel(), dtype=torch.uint8, device="cuda")
            super().pack(bits_, tiles, tmp)
            out.copy_(tmp.cpu())

        def unpack(self, bits_, tiles, buf):
            super().unpack(bits_, tiles, buf.cuda())

    g = api.make_grid(api.map_kind[kind], 3, n, rho)
    side = g.cell_side()
    cells = api.tet_cells(side)
    plan = D.build_plan(g.extents, api.map_outcomes(g), kind == "h3d", g.domain_side(), world)
    sh = D.ShardedLife(plan, rank, rho, StagedOps(g, ex))
    a = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
    b = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
    api.life_init_device(3, side, 42, a)
    b.fill_(1)  # garbage outside owned + halo tiles must never matter
    if engine:  # the per-rank engine: boundary chunks, halo on a comm stream, interior, unpack
        eng = D.ShardedEngine(plan, rank, rho, D.StagedEngineOps(g))
        res = D.engine_launch_ca(eng, api, g, a, api.bits_buffer(g), api.bits_buffer(g), steps)
    elif bits:
        shb = D.ShardedLife(plan, rank, rho, StagedBitsOps(g))
        res = D.run_bits(shb, api, g, a, steps)
    else:
        res = sh.run(a, b, steps)
    torch.cuda.synchronize()
    sh.gather_owned(res, 0)
    if rank == 0:
        orc = Restated()
        want = orc.make_life_state(3, side, 42)
        orc.ca3d_run(side, steps, want)
        q.put(bool((res.cpu().numpy() == want).all()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,rho,ex", [("h3d", 32, 4, 1), ("h3d", 32, 8, 1), ("bb", 31, 4, 1),
                                           ("h3d", 16, 4, 0)])
def test_sharded_step_on_one_gpu(cuda, kind, n, rho, ex):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, n, rho, ex, 4, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok


@pytest.mark.parametrize("kind,n,rho", [("h3d", 32, 4), ("h3d", 32, 8), ("bb", 31, 4), ("h3d", 64, 8)])
def test_sharded_bits_engine_on_one_gpu(cuda, kind, n, rho):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, n, rho, 1, 6, q, True)) for r in range(world)]
    for p in procs:
        p.start()
    ok = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok


def test_bench_sharded_smoke(cuda):
    # bench.py --gpus 2 through torchrun: the sharded bit-shadow engine bench
    # path end to end (gloo + host-staged halo: one GPU cannot host two NCCL ranks)
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SMX_DIST_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus",
                          "2", "--steps", "2", "--warmup", "3"], cwd=root, env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["parity"]["all_cells_equal_passes_once"]
    ca = line["ca_sharded"]["C4"]
    assert "bit-shadow engine" in ca["parallelism"] and ca["value"] > 0
    assert ca["parity"]["ok"] is True, ca["parity"]


def _accum_worker(rank, world, port, kind, n, rho, passes, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2208_11617_b200 import api
    from paper_2208_11617_b200 import dist as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = api.make_grid(api.map_kind[kind], 2, n, rho)
    ex, ey = g.extents[0], g.extents[1]
    ranges = D.partition_rows(D.useful_per_row(api.map_outcomes(g), ex, ey), world)
    cells = torch.zeros(api.tri_cells(g.cell_side()), dtype=torch.int32, device="cuda")
    tot = D.ShardedAccum(g, ranges, rank).run(cells, passes)
    mine = cells.cpu()
    # no cell is touched by two ranks: the shards' states sum to the full result
    dist.all_reduce(mine)
    if rank == 0:
        q.put((bool((mine == passes).all()), tot))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,n,rho", [("h2d", 64, 4), ("bb", 63, 4), ("h2d", 256, 1)])
def test_sharded_accum_rows_on_one_gpu(cuda, kind, n, rho):
    """ACCUM sharded by grid rows over three ranks on cuda:0 (no
    cell data moves, counters all-reduced): every cell = passes exactly once,
    and the summed counters equal one full launch_accum's."""
    from paper_2208_11617_b200 import api
    world, passes = 3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_accum_worker, args=(r, world, port, kind, n, rho, passes, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok, tot = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert ok
    g = api.make_grid(api.map_kind[kind], 2, n, rho)
    rep = api.launch_map_device(g)
    assert (tot["blocks_launched"], tot["blocks_void"], tot["threads_launched"], tot["threads_useful"]) == (
        rep.blocks_launched, rep.blocks_void, rep.threads_launched, rep.threads_useful)


@pytest.mark.parametrize("kind,n,rho,world", [("h3d", 32, 8, 2), ("h3d", 32, 4, 3), ("bb", 31, 8, 2),
                                               ("h3d", 64, 8, 4)])
def test_sharded_engine_on_one_gpu(cuda, kind, n, rho, world):
    """ShardedEngine with the real kernels (plan per wz range, run-list on the
    boundary / interior chunks, bit-tile pack / unpack), ranks on one GPU."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, n, rho, 1, 6, q, False, True))
             for r in range(world)]
    for p in procs:
        p.start()
    ok = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
