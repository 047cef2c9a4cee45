"""Edge cases and limits on the GPU, each against the restated oracle / the
reference: degenerate domains (side 1, one block), rho larger than the block
domain, zero steps, the largest block grid CUDA can launch for H2D at rho = 1
(n = 65536: gridDim.y = 65535), grids beyond the launch limits
(a clean overflow error, not a fault), aliasing and misaligned buffers."""
import numpy as np
import pytest

from oracle.oracle import BB, H2D, H3D, TRAP
from paper_2208_11617_b200 import api

pytestmark = pytest.mark.gpu


def test_degenerate_domains_accum_map(cuda, orc):
    for kind, m, n, rho, T in [(BB, 2, 1, 1, 1), (BB, 3, 1, 1, 1), (H2D, 2, 2, 1, 1), (H3D, 3, 4, 1, 1),
                               (BB, 2, 1, 5, 1), (H2D, 2, 2, 16, 1), (H3D, 3, 4, 7, 1), (TRAP, 2, 2, 3, 1),
                               (TRAP, 2, 3, 1, 16)]:
        g = api.make_grid(kind, m, n, rho, T)
        side = g.cell_side()
        dom = api.simplex_spec(m, side - 1)
        rep = api.launch_map(g, dom)
        cov, cnt = orc.sweep(kind, m, n, rho, T=T)
        assert [rep.blocks_launched, rep.blocks_void, rep.threads_launched, rep.threads_useful] == cnt
        assert (rep.coverage == cov).all() and api.verify_exact_cover(rep, dom).exact
        if m == 2:
            for ex in (api.EXEC_BLOCK, api.EXEC_RUNS):
                st = api.simplex_grid_state(2, side)
                api.launch_accum(g, dom, st, api.launch_opts(exec=ex))
                assert (st.cells == 1).all()


def test_degenerate_life(cuda, orc):
    # side 1 and tiny sides: 3-D dead boundary and 2-D periodic (wraps onto itself)
    for kind, n, rho in [(BB, 1, 1), (H3D, 4, 1), (BB, 2, 1), (BB, 1, 4)]:
        g = api.make_grid(kind, 3, n, rho)
        side = g.cell_side()
        for ex in (api.EXEC_BLOCK,) + ((api.EXEC_RUNS, api.EXEC_BITS) if rho in (4, 8) else ()):
            for alive in (0, 1):
                st = api.simplex_grid_state(3, side, np.uint8, np.full(api.tet_cells(side), alive, np.uint8))
                want = st.cells.copy()
                orc.ca3d_run(side, 3, want)
                api.launch_ca(g, api.simplex_spec(3, side - 1), st,
                              api.launch_opts(steps=3, boundary=api.ca_boundary.dead3d, exec=ex))
                assert (st.cells == want).all(), (kind, n, rho, ex, alive)
    for kind, n, rho in [(BB, 1, 1), (H2D, 2, 1), (BB, 3, 1), (BB, 1, 3)]:
        g = api.make_grid(kind, 2, n, rho)
        side = g.cell_side()
        for ex in (api.EXEC_BLOCK, api.EXEC_RUNS):
            for alive in (0, 1):
                st = api.simplex_grid_state(2, side, np.uint8, np.full(api.tri_cells(side), alive, np.uint8))
                want = st.cells.copy()
                orc.ca2d_run(side, 3, want)
                api.launch_ca(g, api.simplex_spec(2, side - 1), st,
                              api.launch_opts(steps=3, boundary=api.ca_boundary.periodic2d, exec=ex))
                assert (st.cells == want).all(), (kind, n, rho, ex, alive)


def test_zero_steps_and_zero_passes(cuda):
    g = api.make_grid(api.map_kind.h3d, 3, 16, 4)
    side = g.cell_side()
    st = api.make_life_state(3, side, 42)
    h0 = st.hash()
    rep = api.launch_ca(g, api.simplex_spec(3, side - 1), st,
                        api.launch_opts(steps=0, boundary=api.ca_boundary.dead3d))
    assert st.hash() == h0 and rep.state_hash == h0 and rep.blocks_launched == 0
    import torch
    cells = torch.full((api.tri_cells(60),), 7, dtype=torch.int32, device="cuda")
    api.accum_device(api.make_grid(api.map_kind.h2d, 2, 16, 4), cells, passes=0)
    assert int((cells != 7).sum()) == 0


def test_launch_limits_raise_cleanly(cuda):
    import torch
    g = api.make_grid(api.map_kind.h2d, 2, 131072, 1)  # gridDim.y would be 131071 > 65535
    cells = torch.zeros(16, dtype=torch.int32, device="cuda")
    with pytest.raises((api.Overflow, api.InvalidArgument)):
        api.accum_device(g, cells, 1, api.EXEC_BLOCK)
    # aliasing and misaligned device buffers are contract violations, not faults
    g3 = api.make_grid(api.map_kind.h3d, 3, 16, 4)
    n = api.tet_cells(g3.cell_side())
    a = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
    with pytest.raises(api.InvalidArgument):
        api.ca_step_device(g3, a[:n], a[:n], api.EXEC_RUNS)
    with pytest.raises(api.InvalidArgument):
        api.ca_step_device(g3, a[1:n + 1], a[:n], api.EXEC_RUNS)
    torch.cuda.synchronize()


@pytest.mark.slow
def test_h2d_rho1_max_grid_appendix_a(cuda):
    # H2D(65536), rho = 1: 32768 x 65535 blocks (gridDim.y at the CUDA limit),
    # 2,147,450,880 u32 cells; SURVEY Appendix A hash of the one-pass state
    import torch
    g = api.make_grid(api.map_kind.h2d, 2, 65536, 1)
    side = g.cell_side()
    n = api.tri_cells(side)
    for ex in (api.EXEC_RUNS, api.EXEC_BLOCK):
        cells = torch.zeros(n, dtype=torch.int32, device="cuda")
        api.accum_device(g, cells, 1, ex)
        assert int((cells != 1).sum()) == 0, ex
        del cells
        torch.cuda.empty_cache()
    assert api.state_hash(2, side, np.ones(n, np.uint32)) == 8855049223948604461


def test_sequential_kernels_vs_oracle(cuda, orc):
    """kernel_accum / kernel_edm / kernel_ca_run (the reference's sequential
    engines, simulator.hpp:329-331,377-386,402-425) on the GPU, sides that the
    internal tiling handles with the engine (divisible by 8 / 4), the block
    scheme (odd primes, 2 mod 4) and the 2-D periodic rule."""
    st = api.simplex_grid_state(2, 37)
    st.cells[:] = 5
    api.kernel_accum(st)
    assert (st.cells == 6).all()
    for side in (1, 13, 64, 66):
        pts = api.make_edm_points(side, 3)
        st = api.simplex_grid_state(2, side, np.float64)
        api.kernel_edm(pts, st)
        assert (st.cells == orc.kernel_edm(side, 3)).all(), side
    for side in (1, 8, 12, 13, 22, 40):
        st = api.make_life_state(3, side, 42)
        want = st.cells.copy()
        orc.ca3d_run(side, 6, want)
        api.kernel_ca_run(st, 6, api.ca_boundary.dead3d)
        assert (st.cells == want).all(), side
    for side in (7, 16, 63):
        st = api.make_life_state(2, side, 42)
        want = st.cells.copy()
        orc.ca2d_run(side, 9, want)
        api.kernel_ca_run(st, 9, api.ca_boundary.periodic2d)
        assert (st.cells == want).all(), side
