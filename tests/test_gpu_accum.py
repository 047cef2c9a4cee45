"""GPU parity for ACCUM (K2) — H2D and BB, both execution schemes — against the
reference's launch_accum hashes (tests/golden/accum.json) and the oracle."""
import numpy as np
import pytest

from conftest import golden
from oracle.oracle import BB, H2D
from paper_2208_11617_b200 import api

pytestmark = pytest.mark.gpu
EXECS = [api.EXEC_BLOCK, api.EXEC_RUNS]


@pytest.mark.parametrize("ex", EXECS)
def test_accum_hashes_vs_reference(cuda, ex):
    for row in golden("accum.json")["launch_accum"]:
        g = api.make_grid(row["kind"], 2, row["n"], row["rho"])
        side = g.cell_side()
        st = api.simplex_grid_state(2, side)
        rep = api.launch_accum(g, api.simplex_spec(2, side - 1), st,
                               api.launch_opts(record_coverage=False, exec=ex))
        assert rep.state_hash == row["hash"], row
        assert rep.threads_useful == row["threads_useful"]
        if "hash_2pass" in row:
            rep = api.launch_accum(g, api.simplex_spec(2, side - 1), st,
                                   api.launch_opts(record_coverage=False, exec=ex))
            assert rep.state_hash == row["hash_2pass"]


@pytest.mark.parametrize("ex", EXECS)
def test_accum_exact_for_every_pow2_and_rho(cuda, ex):
    # acceptance criterion 3 (n = 2^1..2^12) and the ragged rho cases
    for k in range(1, 13):
        for rho in (1, 3, 16):
            n = 1 << k
            for g in (api.make_grid(api.map_kind.h2d, 2, n, rho), api.make_grid(api.map_kind.bb, 2, n - 1, rho)):
                side = g.cell_side()
                if side < 1:
                    continue
                st = api.simplex_grid_state(2, side)
                rep = api.launch_accum(g, api.simplex_spec(2, side - 1), st, api.launch_opts(exec=ex))
                assert (st.cells == 1).all(), (g, ex)
                assert api.verify_exact_cover(rep, api.simplex_spec(2, side - 1)).exact
                if g.kind == api.map_kind.h2d:
                    assert rep.blocks_void == 0 and rep.blocks_launched == n * (n - 1) // 2


def test_accum_device_multi_pass_and_nonzero_start(cuda):
    import torch
    g = api.make_grid(api.map_kind.h2d, 2, 512, 16)
    n = api.tri_cells(g.cell_side())
    start = torch.randint(0, 1 << 30, (n,), dtype=torch.int32, device="cuda")
    for ex in EXECS:
        cells = start.clone()
        api.accum_device(g, cells, passes=5, exec=ex)
        assert torch.equal(cells, start + 5)


@pytest.mark.slow
def test_c3_full_size_hash(cuda):
    # C3: H2D(4096), rho = 16: 2,146,467,960 u32 cells; one pass -> all ones
    want = {(r["kind"], r["n"], r["rho"]): r["hash"] for r in golden("accum.json")["launch_accum"]}
    import torch
    g = api.make_grid(api.map_kind.h2d, 2, 4096, 16)
    n = api.tri_cells(g.cell_side())
    cells = torch.zeros(n, dtype=torch.int32, device="cuda")
    api.accum_device(g, cells, passes=3, exec=api.EXEC_RUNS)
    assert int((cells != 3).sum()) == 0
    gb = api.make_grid(api.map_kind.bb, 2, 4095, 16)
    api.accum_device(gb, cells, passes=1, exec=api.EXEC_RUNS)
    assert int((cells != 4).sum()) == 0
    del cells
    # Appendix A hash of the one-pass state, computed on the host copy
    host = np.ones(n, np.uint32)
    assert api.state_hash(2, g.cell_side(), host) == 18207742408615288078


def test_pipelined_host_accum(cuda):
    """Host-buffer launch_accum above 512 MB runs pipelined (chunked H2D ||
    map-filtered x-run kernel || D2H); every cell must still be visited exactly
    once, for H2D, BB, padded and trapezoid grids, with the reference's
    counters."""
    rng = np.random.default_rng(1)
    for g in (api.make_grid(api.map_kind.h2d, 2, 1024, 16), api.make_grid(api.map_kind.bb, 2, 1023, 16),
              api.make_grid(api.map_kind.h2d_padded, 2, 1100, 16),
              api.make_grid(api.map_kind.h2d_trapezoid, 2, 1500, 16, 4)):
        side = g.cell_side()
        init = rng.integers(0, 1 << 30, api.tri_cells(side), dtype=np.uint32)
        st = api.simplex_grid_state(2, side, np.uint32, init.copy())
        rep = api.launch_accum(g, api.simplex_spec(2, side - 1), st, api.launch_opts(record_coverage=False))
        assert (st.cells == init + 1).all(), g
        assert rep.threads_useful == api.tri_cells(side)
        assert rep.blocks_launched == g.blocks()
