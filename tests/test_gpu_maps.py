"""GPU parity for the maps (K1) and the MAP kernel: every block's map_outcome is
bit-exact against the reference goldens and the oracle; coverage multisets and
launch counters equal the reference's launch_map."""
import numpy as np
import pytest

from conftest import golden
from oracle.oracle import BB, H2D, H3D
from paper_2208_11617_b200 import api

pytestmark = pytest.mark.gpu


def _kind_grid(kind, m, n):
    return api.grid_h2d(n) if kind == H2D else api.grid_h3d(n) if kind == H3D else api.grid_bb(n, m)


def test_outcomes_bit_exact_vs_reference_goldens(cuda, orc):
    for row in golden("maps.json")["outcomes"]:
        g = _kind_grid(row["kind"], row["m"], row["n"])
        got = api.map_outcomes(g)[:, :6].astype(np.int64)
        assert got.shape[0] == row["blocks"]
        assert orc.state_hash(0, 0, np.ascontiguousarray(got)) == row["hash"], row


def test_c1_coordinate_check_full(cuda, orc):
    # C1: every block of H2D(1024) (523,776) and BB(1023) (1,046,529)
    for kind, m, n in [(H2D, 2, 1024), (BB, 2, 1023), (H3D, 3, 512), (BB, 3, 127)]:
        got = api.map_outcomes(_kind_grid(kind, m, n))[:, :6].astype(np.int64)
        assert (got == orc.map_outcomes(kind, m, n)).all(), (kind, n)


def test_launch_map_counters_and_coverage_vs_reference(cuda, orc):
    for row in golden("maps.json")["launch_map"]:
        g = api.make_grid(row["kind"], row["m"], row["n"], row["rho"])
        side = g.cell_side()
        opts = api.launch_opts(record_coverage="coverage_hash" in row)
        rep = api.launch_map(g, api.simplex_spec(g.dims, side - 1), opts)
        assert [rep.blocks_launched, rep.blocks_void, rep.threads_launched, rep.threads_useful] == [
            row["blocks_launched"], row["blocks_void"], row["threads_launched"], row["threads_useful"]], row
        assert (rep.space_overhead.numerator, rep.space_overhead.denominator) == tuple(row["space_overhead"])
        if "coverage_hash" in row:
            assert orc.state_hash(0, 0, rep.coverage) == row["coverage_hash"], row
            assert api.verify_exact_cover(rep, api.simplex_spec(g.dims, side - 1)).exact == row["all_one"]


def test_h3d_exact_cover_and_ratio_toward_9_8(cuda):
    # acceptance.cpp:127-150 (criterion 5)
    prev = None
    for n in (4, 8, 16, 32, 64, 128):
        g = api.grid_h3d(n)
        rep = api.launch_map(g, api.simplex_spec(3, g.cell_side() - 1))
        assert api.verify_exact_cover(rep, api.simplex_spec(3, g.cell_side() - 1)).exact
        ratio = rep.threads_launched / rep.threads_useful
        assert ratio > 1.125
        if prev is not None:
            assert ratio < prev
        prev = ratio
    assert abs(prev - 1.125) / 1.125 < 0.10
    assert (rep.threads_launched, rep.threads_useful) == (6144 * 64, 5461 * 64)


def test_h2d_slack_bound(cuda):
    # acceptance.cpp:262-279 (criterion 9)
    for rho, want in [(2, 1023), (4, 6138), (8, 28644), (16, 122760)]:
        g = api.make_grid(api.map_kind.h2d, 2, 1024, rho)
        rep = api.launch_map(g, api.simplex_spec(2, g.cell_side() - 1), api.launch_opts(record_coverage=False))
        assert rep.threads_launched - rep.threads_useful == want


def test_cover_verdict_pinpoints_planted_defect(cuda):
    # test_simulator.cpp:324-338
    g = api.grid_h2d(16)
    dom = api.simplex_spec(2, g.cell_side() - 1)
    rep = api.launch_map(g, dom)
    assert api.verify_exact_cover(rep, dom).exact
    rep.coverage[api.tri_linear_index(2, 5)] -= 1
    rep.coverage[api.tri_linear_index(3, 7)] += 1
    v = api.verify_exact_cover(rep, dom)
    assert not v.exact and v.witness == api.data_coord(2, 5, 0) and v.multiplicity == 0


def test_map_kernel_runs(cuda):
    import torch
    for g in (api.grid_h2d(1024), api.grid_bb(1023, 2), api.grid_h3d(256), api.grid_bb(255, 3)):
        api.map_kernel_device(g)
    torch.cuda.synchronize()
