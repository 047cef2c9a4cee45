"""The CPU oracle, pinned before it is trusted (CPU suite).

1. the restatement (oracle/smx_oracle.c) against the golden vectors generated
   by the reference itself (tests/golden/*.json, gen_golden.py);
2. against the values the reference's own tests pin (test_maps.cpp,
   test_simulator.cpp, acceptance.cpp);
3. against oracle/_ref directly on seeded inputs when it is built.
"""
import numpy as np
import pytest

from conftest import golden
from oracle.oracle import BB, H2D, H3D, cells_of


def test_map_outcomes_match_reference_goldens(orc):
    for row in golden("maps.json")["outcomes"]:
        o = orc.map_outcomes(row["kind"], row["m"], row["n"])
        assert o.shape[0] == row["blocks"]
        assert int(o[:, 0].sum()) == row["voids"]
        assert orc.state_hash(0, 0, o) == row["hash"], row


def test_tiny_outcome_arrays(orc):
    for row in golden("maps.json")["tiny"]:
        o = orc.map_outcomes(row["kind"], row["m"], row["n"])
        assert o.tolist() == row["outcomes"]


def test_pinned_points_from_reference_tests(orc):
    # test_maps.cpp:123-128, :244
    assert orc.map_one(H2D, 2, 0, 0, 0)[1:3] == (0, 1)
    assert orc.map_one(H2D, 2, 0, 3, 0)[1:3] == (6, 7)
    assert orc.map_one(H2D, 2, 0, 2, 1)[1:3] == (4, 6)
    assert orc.map_one(H2D, 2, 0, 1, 2)[1:3] == (1, 3)
    assert orc.map_one(H2D, 2, 0, 2, 1)[4:6] == (2, 1)
    assert orc.map_one(H3D, 3, 8, 0, 0, 0)[1:4] == (0, 5, 0)
    # test_maps.cpp:41-47 (bb)
    assert orc.map_one(BB, 2, 8, 1, 3, 0)[:4] == (0, 1, 3, 0)
    assert orc.map_one(BB, 2, 8, 7, 2, 0)[0] == 1


def test_h3d_void_counts_pinned(orc):
    # test_maps.cpp:247: {2, 12, 88, 688, 5472} for n = 4..64
    for n, v in zip([4, 8, 16, 32, 64], [2, 12, 88, 688, 5472]):
        assert int(orc.map_outcomes(H3D, 3, n)[:, 0].sum()) == v
    # grid shapes (test_maps.cpp:113-118, :237-238)
    assert orc.grid(H3D, 3, 4) == (2, 2, 3)
    ex, ey, ez = orc.grid(H3D, 3, 64)
    assert ex * ey * ez == 49152
    ex, ey, _ = orc.grid(H2D, 2, 1024)
    assert ex * ey == 523776


def test_sweep_counters_and_coverage_match_reference(orc):
    for row in golden("maps.json")["launch_map"]:
        if row["threads_launched"] > 40_000_000:
            continue
        cov, cnt = orc.sweep(row["kind"], row["m"], row["n"], row["rho"], coverage="coverage_hash" in row)
        assert cnt == [row["blocks_launched"], row["blocks_void"], row["threads_launched"],
                       row["threads_useful"]], row
        if "coverage_hash" in row:
            assert orc.state_hash(0, 0, cov) == row["coverage_hash"]
            assert bool((cov == 1).all()) == row["all_one"]


def test_bb_accounting_pinned():
    # test_simulator.cpp:93-109 and acceptance.cpp:66-88 via the golden rows
    rows = {(r["kind"], r["m"], r["n"], r["rho"]): r for r in golden("maps.json")["launch_map"]}
    r = rows[(BB, 2, 4, 1)]
    assert (r["blocks_launched"], r["blocks_void"], r["threads_useful"]) == (16, 6, 10)
    assert r["space_overhead"] == [3, 5]
    assert rows[(BB, 3, 4, 1)]["space_overhead"] == [11, 5]
    # SURVEY §8(d) exact rationals
    assert rows[(H2D, 2, 1024, 16)]["space_overhead"] == [15, 16369]
    assert rows[(BB, 2, 1023, 16)]["space_overhead"] == [16367, 16369]
    assert rows[(H3D, 3, 64, 4)]["space_overhead"] == [37227, 224917]
    assert rows[(BB, 3, 63, 4)]["space_overhead"] == [158381, 32131]
    assert rows[(H3D, 3, 128, 8)]["space_overhead"] == [1083949, 7304659]
    assert rows[(BB, 3, 127, 8)]["space_overhead"] == [859705, 172551]
    # slack (n-1) rho (rho-1) / 2 (acceptance.cpp:262-279)
    for rho in (2, 4):
        r = rows[(H2D, 2, 64, rho)]
        assert r["threads_launched"] - r["threads_useful"] == 63 * rho * (rho - 1) // 2


def test_accum_hashes_match_reference(orc):
    for row in golden("accum.json")["launch_accum"]:
        side = (row["n"] if row["kind"] == BB else row["n"] - 1) * row["rho"]
        if cells_of(2, side) > 50_000_000:
            continue
        cells = np.zeros(cells_of(2, side), np.uint32)
        _, cnt = orc.sweep(row["kind"], 2, row["n"], row["rho"], coverage=False, cells=cells)
        assert orc.state_hash(2, side, cells) == row["hash"], row
        assert cnt[3] == row["threads_useful"]


def test_accum_appendix_a():
    rows = {(r["kind"], r["n"], r["rho"]): r["hash"] for r in golden("accum.json")["launch_accum"]}
    assert rows[(H2D, 1024, 1)] == 9376064259860285065
    assert rows[(H2D, 1024, 16)] == 625406489163772878
    assert rows[(H2D, 4096, 1)] == 3142058413832162077


def test_life_init_matches_reference(orc):
    for row in golden("ca.json")["life_init"]:
        if cells_of(row["m"], row["side"]) > 200_000_000:
            continue
        s = orc.make_life_state(row["m"], row["side"], row["seed"])
        assert orc.state_hash(row["m"], row["side"], s) == row["hash"], row
        assert int(s.sum()) == row["alive"]


def test_fast_ca_matches_reference_goldens(orc):
    for row in golden("ca.json")["kernel_ca_run"]:
        s = orc.make_life_state(3, row["side"], row["seed"])
        orc.ca3d_run(row["side"], row["steps"], s)
        assert orc.state_hash(3, row["side"], s) == row["hash"], row
        assert int(s.sum()) == row["alive"]


def test_literal_ca_matches_fast_ca(orc):
    for side, steps, seed in [(6, 3, 0), (7, 6, 11), (13, 5, 2), (20, 4, 42)]:
        a = orc.make_life_state(3, side, seed)
        b = a.copy()
        orc.ca3d_run(side, steps, a)
        orc.ca3d_run_literal(side, steps, b)
        assert (a == b).all()


def test_ca_appendix_a_hashes():
    rows = {(r["side"], r["steps"], r["seed"]): r for r in golden("ca.json")["kernel_ca_run"]}
    assert rows[(15, 64, 42)]["hash"] == 750086803756986311
    assert rows[(31, 64, 42)]["hash"] == 11768087780779516714
    assert rows[(63, 64, 42)]["hash"] == 6734372989930245576
    assert rows[(63, 100, 42)]["hash"] == 14612348930500829140
    assert rows[(127, 8, 42)]["hash"] == 17112464122791685253
    assert rows[(255, 1, 42)]["hash"] == 13808704447608628426
    assert rows[(255, 2, 42)]["hash"] == 8192526562866132158


def test_launch_ca_rows_equal_sequential(orc):
    # launch_ca through H3D/BB grids == kernel_ca_run on the same cell side
    for row in golden("ca.json")["launch_ca"]:
        s = orc.make_life_state(3, row["side"], row["seed"])
        orc.ca3d_run(row["side"], row["steps"], s)
        assert orc.state_hash(3, row["side"], s) == row["hash"], row


def test_dead_boundary_starves_lone_cell(orc):
    # test_simulator.cpp:311-316
    side = 6
    s = np.zeros(cells_of(3, side), np.uint8)
    s[int(orc.L.orc_tet_layer_prefix(side, 1)) + 2 * 3 // 2 + 1] = 1  # (1, 2, 1)
    orc.ca3d_run(side, 1, s)
    assert int(s.sum()) == 0


@pytest.mark.parametrize("kind,m,n", [(H2D, 2, 64), (H3D, 3, 32), (BB, 3, 9), (BB, 2, 33)])
def test_restated_maps_equal_reference_directly(ref, orc, kind, m, n):
    assert (ref.map_outcomes(kind, m, n) == orc.map_outcomes(kind, m, n)).all()


def test_restated_ca_equals_reference_directly(ref, orc):
    for side, steps, seed in [(9, 7, 123), (17, 3, 9)]:
        a = ref.make_life_state(3, side, seed)
        b = orc.make_life_state(3, side, seed)
        assert (a == b).all()
        ref.kernel_ca_run(3, side, steps, a)
        orc.ca3d_run(side, steps, b)
        assert (a == b).all()


def test_full_size_goldens_small_cases(orc):
    """tests/golden/ca_full.json (gen_golden_full.py): the cases cheap enough
    to recompute here — the exact C2 bench tuple (side 252, 100 steps) and the
    reference's own side-1023 one-step hash."""
    from conftest import golden
    cases = golden("ca_full.json")["cases"]
    for key in ("c2_rho4_100", "side1023_1"):
        c = cases[key]
        s = orc.make_life_state(3, c["side"], 42)
        assert orc.state_hash(3, c["side"], s) == int(c["init_hash"])
        orc.ca3d_run(c["side"], c["steps"], s)
        assert orc.state_hash(3, c["side"], s) == int(c["final_hash"]), key
    assert int(cases["side1023_1"]["final_hash"]) == 13036985295180606544


def test_reference_accum_sample(ref):
    """The bench's reference arm: the reference's own launch_accum sweep over
    the first block rows of a grid, concurrent replicas."""
    from oracle.oracle import H2D
    secs, useful = ref.accum_sample(H2D, 2, 64, 4, 8, 2, 0, 2)
    assert len(secs) == 2 and all(s > 0 for s in secs)
    # first 8 block rows of H2D(64) (ex = 32), rho = 4: count their member
    # cells from the restated map outcomes (strict view: y - 1)
    from oracle.oracle import Restated
    out = Restated().map_outcomes(H2D, 2, 64)[: 32 * 8]
    side, want = 63 * 4, 0
    for o in out:
        if o[0]:
            continue
        bx, by = o[1] * 4, (o[2] - 1) * 4
        want += sum(1 for ly in range(4) for lx in range(4) if bx + lx <= by + ly < side)
    assert useful == want
