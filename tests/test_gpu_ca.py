"""GPU parity for Life init (K4) and the 3-D dead-boundary CA step (K3), H3D and
BB, both execution schemes, against the reference goldens and the oracle."""
import numpy as np
import pytest

from conftest import golden
from oracle.oracle import BB, H3D
from paper_2208_11617_b200 import api

pytestmark = pytest.mark.gpu


def run_gpu(g, side, seed, steps, ex):
    st = api.make_life_state(3, side, seed)
    api.launch_ca(g, api.simplex_spec(3, side - 1), st,
                  api.launch_opts(steps=steps, boundary=api.ca_boundary.dead3d, exec=ex, record_coverage=False))
    return st


def test_life_init_vs_reference(cuda):
    for row in golden("ca.json")["life_init"]:
        st = api.make_life_state(row["m"], row["side"], row["seed"])
        assert st.hash() == row["hash"], row
        assert int(st.cells.sum(dtype=np.int64)) == row["alive"]


XRUN = (api.EXEC_RUNS, api.EXEC_BITS)  # fused u8 step, bit-shadow engine
ALL_EX = (api.EXEC_BLOCK,) + XRUN


@pytest.mark.parametrize("ex", ALL_EX)
def test_launch_ca_rows_vs_reference(cuda, ex):
    for row in golden("ca.json")["launch_ca"]:
        if ex in XRUN and row["rho"] not in (4, 8):
            continue
        g = api.make_grid(row["kind"], 3, row["n"], row["rho"])
        st = run_gpu(g, row["side"], row["seed"], row["steps"], ex)
        assert st.hash() == row["hash"], row


def test_appendix_a_hashes(cuda):
    # rho = 1 grids (block scheme) over sides 15..255
    rows = {(r["side"], r["steps"], r["seed"]): r["hash"] for r in golden("ca.json")["kernel_ca_run"]}
    for side, steps in [(15, 64), (31, 64), (63, 64), (63, 100), (127, 8), (255, 1), (255, 2)]:
        for g in (api.grid_h3d(side + 1), api.grid_bb(side, 3)):
            st = run_gpu(g, side, 42, steps, api.EXEC_BLOCK)
            assert st.hash() == rows[(side, steps, 42)], (g, side, steps)


@pytest.mark.parametrize("kind", [H3D, BB])
@pytest.mark.parametrize("rho", [4, 8])
def test_runs_scheme_vs_oracle_many_steps(cuda, orc, kind, rho):
    for n in ([8, 16, 32, 64] if kind == H3D else [7, 15, 31, 63]):
        g = api.make_grid(kind, 3, n, rho)
        side = g.cell_side()
        steps = 5
        want = orc.make_life_state(3, side, 7)
        orc.ca3d_run(side, steps, want)
        for ex in ALL_EX:
            got = run_gpu(g, side, 7, steps, ex)
            assert (got.cells == want).all(), (kind, n, rho, ex)


def test_block_scheme_odd_rho(cuda, orc):
    for kind, n, rho in [(H3D, 8, 3), (H3D, 4, 5), (BB, 5, 3), (H3D, 16, 2), (BB, 9, 6), (H3D, 8, 16)]:
        g = api.make_grid(kind, 3, n, rho)
        side = g.cell_side()
        want = orc.make_life_state(3, side, 3)
        orc.ca3d_run(side, 4, want)
        got = run_gpu(g, side, 3, 4, api.EXEC_BLOCK)
        assert (got.cells == want).all(), (kind, n, rho)


def test_dense_random_states(cuda, orc):
    # not just the 1/4-density init: dense and sparse random states, 1 step
    import torch
    rng = np.random.default_rng(5)
    for kind, n, rho in [(H3D, 32, 4), (BB, 31, 4), (H3D, 16, 8), (BB, 15, 8)]:
        g = api.make_grid(kind, 3, n, rho)
        side = g.cell_side()
        for p in (0.05, 0.5, 0.95):
            init = (rng.random(api.tet_cells(side)) < p).astype(np.uint8)
            want = init.copy()
            orc.ca3d_run(side, 1, want)
            for ex in ALL_EX:
                cur = torch.from_numpy(init).cuda()
                nxt = torch.empty_like(cur)
                api.ca_step_device(g, cur, nxt, ex)
                assert (nxt.cpu().numpy() == want).all(), (kind, n, rho, p, ex)


def test_ca_counters_and_coverage(cuda):
    rows = {(r["kind"], r["n"], r["rho"]): r for r in golden("ca.json")["launch_ca"]}
    for (kind, n, rho), row in rows.items():
        g = api.make_grid(kind, 3, n, rho)
        side = g.cell_side()
        st = api.make_life_state(3, side, 42)
        rep = api.launch_ca(g, api.simplex_spec(3, side - 1), st,
                            api.launch_opts(steps=1, boundary=api.ca_boundary.dead3d))
        assert (rep.blocks_launched, rep.blocks_void, rep.threads_useful) == (
            row["blocks_launched"], row["blocks_void"], row["threads_useful"])
        assert api.verify_exact_cover(rep, api.simplex_spec(3, side - 1)).exact


@pytest.mark.slow
def test_c4_100_steps_vs_restated_oracle(cuda, orc):
    # C4: H3D(128), rho = 8, side 1016 (175,311,816 cells), 100 steps, seed 42
    import torch
    g = api.make_grid(api.map_kind.h3d, 3, 128, 8)
    side = g.cell_side()
    n = api.tet_cells(side)
    cur = torch.empty(n, dtype=torch.uint8, device="cuda")
    api.life_init_device(3, side, 42, cur)
    want = orc.make_life_state(3, side, 42)
    assert (cur.cpu().numpy() == want).all()
    api.ca_device(g, cur, 100, api.EXEC_RUNS)
    orc.ca3d_run(side, 100, want)
    got = cur.cpu().numpy()
    assert api.state_hash(3, side, got) == api.state_hash(3, side, want)
    # BB over the same domain agrees too
    gb = api.make_grid(api.map_kind.bb, 3, 127, 8)
    api.life_init_device(3, side, 42, cur)
    api.ca_device(gb, cur, 100, api.EXEC_RUNS)
    assert (cur.cpu().numpy() == want).all()
    # and the product path: the bit-shadow engine (pack, plan, one persistent
    # launch of all 100 steps, unpack), H and BB
    for grid in (g, gb):
        api.life_init_device(3, side, 42, cur)
        api.ca_device(grid, cur, 100, api.EXEC_BITS)
        assert (cur.cpu().numpy() == want).all(), grid


@pytest.mark.slow
def test_c5_full_size_engine_vs_block_scheme(cuda):
    """C5: H3D(256), rho = 8, side 2040 (1,417,025,480 cells). The engine's
    3 steps (H3D and BB) equal 3 steps of the paper's one-thread-per-cell block
    scheme (an independent kernel: 26 byte neighbours through L1), and one
    single-step u8 -> u8 call equals one block step; compared on the device."""
    import torch
    g = api.make_grid(api.map_kind.h3d, 3, 256, 8)
    gb = api.make_grid(api.map_kind.bb, 3, 255, 8)
    side = g.cell_side()
    n = api.tet_cells(side)
    a = torch.empty(n + 256, dtype=torch.uint8, device="cuda")[:n]
    b = torch.empty(n + 256, dtype=torch.uint8, device="cuda")[:n]
    ref = torch.empty(n + 256, dtype=torch.uint8, device="cuda")[:n]
    api.life_init_device(3, side, 42, ref)
    for _ in range(3):  # block scheme, u8 -> u8 per step
        api.ca_step_device(g, ref, b, api.EXEC_BLOCK)
        ref, b = b, ref
    for grid in (g, gb):
        api.life_init_device(3, side, 42, a)
        api.ca_device(grid, a, 3, api.EXEC_BITS)
        assert torch.equal(a, ref), grid
    api.life_init_device(3, side, 42, a)
    api.ca_step_device(g, a, b, api.EXEC_AUTO)
    api.life_init_device(3, side, 42, ref)
    api.ca_step_device(gb, ref, a, api.EXEC_BLOCK)
    assert torch.equal(a, b)
