"""GPU parity for the general-n and comparison 2-D maps:
H padded, concurrent trapezoids (one launch per band), RB and lambda — block
outcomes bit-exact against the reference goldens and the restated oracle;
launch_map counters / exact space_overhead / coverage and launch_accum state
hashes equal to the reference's (tests/golden/maps2d.json); every n up to 512
tiled exactly by its trapezoid bands; general-n ACCUM at the C3 scale."""
import numpy as np
import pytest

from conftest import golden
from oracle.oracle import TRAP
from paper_2208_11617_b200 import api

pytestmark = pytest.mark.gpu
G = golden("maps2d.json")


def _grid(kind, n, rho=1, T=1):
    return api.make_grid(kind, 2, n, rho, T)


def test_outcomes_bit_exact(cuda, orc):
    for row in G["outcomes"]:
        got = api.map_outcomes(_grid(row["kind"], row["n"], 1, row["T"]))[:, :6].astype(np.int64)
        assert got.shape[0] == row["blocks"], row
        assert orc.state_hash(0, 0, np.ascontiguousarray(got)) == row["hash"], row
        assert (got == orc.map_outcomes(row["kind"], 2, row["n"], row["T"])).all(), row


def test_launch_map_vs_reference(cuda, orc):
    for row in G["launch_map"]:
        g = _grid(row["kind"], row["n"], row["rho"], row["T"])
        dom = api.simplex_spec(2, g.cell_side() - 1)
        rep = api.launch_map(g, dom)
        assert [rep.blocks_launched, rep.blocks_void, rep.threads_launched, rep.threads_useful] == [
            row["blocks_launched"], row["blocks_void"], row["threads_launched"], row["threads_useful"]], row
        assert (rep.space_overhead.numerator, rep.space_overhead.denominator) == tuple(row["space_overhead"])
        assert orc.state_hash(0, 0, rep.coverage) == row["coverage_hash"], row
        assert api.verify_exact_cover(rep, dom).exact == row["all_one"]


@pytest.mark.parametrize("ex", [api.EXEC_BLOCK, api.EXEC_RUNS])
def test_launch_accum_vs_reference(cuda, ex):
    for row in G["launch_accum"]:
        g = _grid(row["kind"], row["n"], row["rho"], row["T"])
        st = api.simplex_grid_state(2, g.cell_side())
        rep = api.launch_accum(g, api.simplex_spec(2, g.cell_side() - 1), st,
                               api.launch_opts(exec=ex, record_coverage=False))
        assert st.hash() == row["hash"], (row, ex)
        assert rep.threads_useful == row["threads_useful"] and rep.blocks_void == row["blocks_void"]


def test_trapezoid_union_tiles_every_n(cuda):
    # test_maps.cpp:222-234 on the GPU: every n in [2, 512], T in {1, 4, 16}
    for n in range(2, 513):
        for T in (1, 4, 16):
            g = api.grid_trapezoids(n, T)
            assert len(g.traps) <= max(1, (n - 1).bit_length())
            dom = api.simplex_spec(2, g.cell_side() - 1)
            rep = api.launch_map(g, dom)
            assert api.verify_exact_cover(rep, dom).exact, (n, T)
            assert rep.threads_useful == api.tri_cells(n - 1)


def test_padded_general_n_exact(cuda):
    # test_maps.cpp:146-165 on the GPU
    for n in (2, 3, 5, 27, 100, 255, 257, 1000, 4097):
        g = api.grid_h2d_padded(n)
        dom = api.simplex_spec(2, g.cell_side() - 1)
        rep = api.launch_map(g, dom)
        assert api.verify_exact_cover(rep, dom).exact
        assert rep.blocks_launched == g.blocks() and rep.blocks_launched - rep.blocks_void == api.tri_cells(n - 1)


def test_general_n_accum_c3_scale(cuda, orc):
    # a non-power-of-two side at the C3 scale: trapezoids n = 4097 (bands
    # 4096 + padded tail), rho = 16 -> side 65536, 2,147,516,416 u32 cells;
    # one pass must leave every cell at exactly 1 (exact cover), counters exact
    import torch
    g = api.make_grid(api.map_kind.h2d_trapezoid, 2, 4097, 16, 4)
    side = g.cell_side()
    cells = torch.zeros(api.tri_cells(side), dtype=torch.int32, device="cuda")
    api.accum_device(g, cells, 1, api.EXEC_RUNS)
    assert int((cells != 1).sum().item()) == 0
    rep = api.launch_map_device(g)
    _, cnt = orc.sweep(TRAP, 2, 4097, 1, coverage=False, T=4)
    assert rep.blocks_launched == cnt[0] and rep.blocks_void == cnt[1]
    assert rep.threads_useful == api.tri_cells(side)


# ---- EDM and periodic 2-D Life (#3) through every 2-D map ----

def _side(kind, n, rho):
    return (n - 1 if api.strict_view(kind) else n) * rho


@pytest.mark.parametrize("ex", [api.EXEC_BLOCK, api.EXEC_RUNS])
def test_edm_bit_exact_vs_reference(cuda, ex):
    # test_simulator.cpp:199-228: launch_edm through every map == the sequential fill
    E = G["edm"]
    for row in E["launch_edm"]:
        g = _grid(row["kind"], row["n"], row["rho"], row["T"])
        side = g.cell_side()
        pts = api.make_edm_points(side, row["seed"])
        st = api.simplex_grid_state(2, side, np.float64)
        rep = api.launch_edm(g, api.simplex_spec(2, side - 1), pts, st,
                             api.launch_opts(exec=ex, record_coverage=False))
        assert st.hash() == row["hash"] and rep.state_hash == row["hash"], (row, ex)
        assert rep.threads_useful == row["threads_useful"]
    # acceptance.cpp:182-200 (criterion 7): sides 63, 255, 1023, two seeds, the five maps
    seq = {(r["side"], r["seed"]): r["hash"] for r in E["kernel_edm"]}
    for side in (63, 255, 1023):
        for seed in (42, 0xC0FFEE):
            pts = api.make_edm_points(side, seed)
            for g in (api.grid_bb(side, 2), api.grid_rb(side), api.grid_lambda(side), api.grid_h2d(side + 1)
                      if side + 1 in (64, 256, 1024) else None, api.grid_trapezoids(side + 1, 1)):
                if g is None:
                    continue
                st = api.simplex_grid_state(2, side, np.float64)
                api.launch_edm(g, api.simplex_spec(2, side - 1), pts, st, api.launch_opts(exec=ex,
                                                                                           record_coverage=False))
                assert st.hash() == seq[(side, seed)], (side, seed, g, ex)


def test_edm_c1_scale_vs_restated(cuda, orc):
    # H2D(1024), rho = 16: side 16368, 133,963,896 f64 cells (1.07 GB), bit-exact
    import torch
    g = api.make_grid(api.map_kind.h2d, 2, 1024, 16)
    side = g.cell_side()
    pts = torch.from_numpy(api.make_edm_points(side, 42)).cuda()
    cells = torch.empty(api.tri_cells(side), dtype=torch.float64, device="cuda")
    api.edm_device(g, pts, cells, api.EXEC_RUNS)
    want = orc.kernel_edm(side, 42)
    assert orc.state_hash(2, side, cells.cpu().numpy()) == orc.state_hash(2, side, want)


@pytest.mark.parametrize("ex", [api.EXEC_BLOCK, api.EXEC_RUNS])
def test_ca2d_periodic_vs_reference(cuda, ex):
    C2 = G["ca2d"]
    for row in C2["life_init"]:
        st = api.make_life_state(2, row["side"], row["seed"])
        assert st.hash() == row["hash"] and int(st.cells.sum()) == row["alive"]
    for row in C2["launch_ca"]:
        g = _grid(row["kind"], row["n"], row["rho"], row["T"])
        st = api.make_life_state(2, row["side"], row["seed"])
        rep = api.launch_ca(g, api.simplex_spec(2, row["side"] - 1), st,
                            api.launch_opts(steps=row["steps"], boundary=api.ca_boundary.periodic2d, exec=ex,
                                            record_coverage=False))
        assert rep.state_hash == row["hash"], (row, ex)
        assert rep.threads_useful == row["threads_useful"]
    # acceptance.cpp:182-205 + SURVEY Appendix A: 64 steps, every map, sides 63..1023
    seq = {(r["side"], r["steps"], r["seed"]): r["hash"] for r in C2["kernel_ca_run"]}
    for side, seed in ((63, 42), (255, 42), (1023, 42), (255, 0xC0FFEE)):
        for g in (api.grid_bb(side, 2), api.grid_rb(side), api.grid_lambda(side), api.grid_h2d(side + 1)
                  if side + 1 in (64, 256, 1024) else None, api.grid_trapezoids(side + 1, 1)):
            if g is None:
                continue
            st = api.make_life_state(2, side, seed)
            api.launch_ca(g, api.simplex_spec(2, side - 1), st,
                          api.launch_opts(steps=64, boundary=api.ca_boundary.periodic2d, exec=ex,
                                          record_coverage=False))
            assert st.hash() == seq[(side, 64, seed)], (side, seed, g, ex)


def test_ca2d_runs_every_small_side_vs_restated(cuda, orc):
    """The bit-sliced x-run 2-D Life kernel against the restated oracle for every
    side 1..80 and rho in {1, 3, 8, 16, 32} (odd alignments of every packed
    row, the wrap rows 0 / S-2 / S-1, runs shorter and longer than one 32-cell
    item), through H, BB, RB and trapezoid grids; 3 steps each."""
    import torch
    def run(g, init):
        a = torch.from_numpy(init.copy()).cuda()
        b = torch.empty_like(a)
        for _ in range(3):
            api.ca_step_device(g, a, b, api.EXEC_RUNS)
            a, b = b, a
        return a.cpu().numpy()

    for side in range(1, 81):
        init = orc.make_life_state(2, side, 1000 + side)
        want = orc.ca2d_run(side, 3, init.copy())
        for rho in (1, 3, 8, 16, 32):
            if side % rho == 0:
                for kind in (api.map_kind.bb, api.map_kind.rb):
                    g = api.make_grid(kind, 2, side // rho, rho)
                    assert np.array_equal(run(g, init), want), (side, rho, g)
    for side in range(1, 81):
        init = orc.make_life_state(2, side, 7 * side)
        want = orc.ca2d_run(side, 3, init.copy())
        grids = [api.grid_trapezoids(side + 1, 4), api.grid_lambda(side)]
        n = side + 1
        if n & (n - 1) == 0 and n >= 2:
            grids.append(api.grid_h2d(n))
        for g in grids:
            assert np.array_equal(run(g, init), want), (side, g)


def test_ca2d_runs_large_rho16_vs_block(cuda):
    """F3's shape (H2D n=1024, rho=16, side 16368): one RUNS step equals one
    BLOCK step cell for cell, and the same for BB over the same domain."""
    import torch
    gh = api.make_grid(api.map_kind.h2d, 2, 1024, 16)
    gb = api.make_grid(api.map_kind.bb, 2, 1023, 16)
    side = gh.cell_side()
    a = torch.empty(api.tri_cells(side), dtype=torch.uint8, device="cuda")
    api.life_init_device(2, side, 42, a)
    r1, r2, r3 = torch.empty_like(a), torch.empty_like(a), torch.empty_like(a)
    api.ca_step_device(gh, a, r1, api.EXEC_RUNS)
    api.ca_step_device(gh, a, r2, api.EXEC_BLOCK)
    api.ca_step_device(gb, a, r3, api.EXEC_RUNS)
    assert torch.equal(r1, r2) and torch.equal(r1, r3)
