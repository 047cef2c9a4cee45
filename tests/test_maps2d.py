"""General-n and comparison 2-D maps (H padded,
concurrent trapezoids, RB, lambda) on the CPU: the restated oracle against the
reference goldens (tests/golden/maps2d.json, generated from oracle/_ref), the
reference's own pinned values (test_maps.cpp:146-234, acceptance.cpp:108-125),
and the C ABI's host-side map arithmetic (include/smx_maps.hpp, the same code
the kernels inline) against the restatement. No GPU needed."""
import numpy as np
import pytest

from conftest import golden
from oracle.oracle import H2D, LAMBDA, PADDED, RB, TRAP
from paper_2208_11617_b200 import api

G = golden("maps2d.json")


def _side(kind, n, rho):
    return (n - 1 if kind in (PADDED, TRAP, H2D) else n) * rho


def test_restated_outcomes_vs_reference_goldens(orc):
    for row in G["outcomes"]:
        o = orc.map_outcomes(row["kind"], 2, row["n"], row["T"])
        assert o.shape[0] == row["blocks"] and int(o[:, 0].sum()) == row["voids"], row
        assert orc.state_hash(0, 0, o) == row["hash"], row


def test_restated_decompositions_vs_reference(orc):
    for row in G["decompositions"]:
        assert orc.decompose_trapezoids(row["n"], row["T"]) == row["bands"], row


def test_restated_sweep_vs_reference_launch_map_and_accum(orc):
    for row in G["launch_map"]:
        cov, cnt = orc.sweep(row["kind"], 2, row["n"], row["rho"], T=row["T"])
        assert cnt == [row["blocks_launched"], row["blocks_void"], row["threads_launched"],
                       row["threads_useful"]], row
        assert orc.state_hash(0, 0, cov) == row["coverage_hash"], row
    for row in G["launch_accum"]:
        side = _side(row["kind"], row["n"], row["rho"])
        cells = np.zeros(side * (side + 1) // 2, np.uint32)
        orc.sweep(row["kind"], 2, row["n"], row["rho"], coverage=False, cells=cells, T=row["T"])
        assert orc.state_hash(2, side, cells) == row["hash"], row


def test_abi_decomposition_matches_golden_and_restated(orc):
    for row in G["decompositions"]:
        got = [vars(t) for t in api.decompose_trapezoids(row["n"], row["T"])]
        assert got == row["bands"], row
    for n in range(2, 700):
        for T in (1, 2, 4, 16):
            assert [vars(t) for t in api.decompose_trapezoids(n, T)] == orc.decompose_trapezoids(n, T)


def test_reference_pinned_values():
    # test_maps.cpp:146-169
    assert api.grid_h2d_padded(8).extents == api.grid_h2d(8).extents
    assert api.grid_h2d_padded(9).extents == (8, 15, 1)
    g = api.grid_h2d_padded(257)
    assert 3.9 < g.blocks() / api.tri_cells(256) < 4.1
    # test_maps.cpp:171-200
    for T in (1, 4, 16):
        t = api.decompose_trapezoids(16, T)
        assert len(t) == 1 and t[0].band == 16 and t[0].h2 == 0 and t[0].valid_side == 16
        assert (t[0].ext_x, t[0].ext_y) == api.grid_h2d(16).extents[:2]
    t27 = api.decompose_trapezoids(27, 1)
    assert [(t.delta_x, t.band, t.h2) for t in t27] == [(0, 16, 11), (16, 8, 3), (24, 2, 1)]
    assert all(t.h1 + t.h2 == t.ext_y - 1 for t in t27)
    t27p = api.decompose_trapezoids(27, 4)
    assert len(t27p) == 3 and (t27p[2].band, t27p[2].h2, t27p[2].valid_side) == (4, 0, 3)
    # test_maps.cpp:202-220: pinned boundary blocks, out-of-grid throws, band == map_h2d
    assert api.map_h2d_trapezoid(api.data_coord(0, 25, 0), 27, 1, 0).target == api.data_coord(0, 26, 0)
    assert api.map_h2d_trapezoid(api.data_coord(0, 26, 0), 27, 1, 0).target == api.data_coord(8, 16, 0)
    with pytest.raises(api.InvalidArgument):
        api.map_h2d_trapezoid(api.data_coord(0, 37, 0), 27, 1, 0)
    single = api.decompose_trapezoids(32, 1)
    assert len(single) == 1
    for oy in range(single[0].ext_y):
        for ox in range(single[0].ext_x):
            w = api.data_coord(ox, oy, 0)
            assert api.map_h2d_trapezoid(w, 32, 1, 0).target == api.map_h2d(w).target


def test_abi_host_maps_match_restated(orc):
    for n in (1, 2, 3, 8, 27, 64):
        ex, ey, _ = api.grid_rb(n).extents
        for y in range(ey):
            for x in range(ex):
                t = api.map_rb_2d(api.data_coord(x, y, 0), n)
                assert (0, t.x, t.y, 0, 1, 0) == orc.map_one(RB, 2, n, x, y), (n, x, y)
    for n in (1, 5, 40):
        for i in range(api.tri_cells(n)):
            t = api.map_lambda_2d(i, n)
            assert (0, t.x, t.y, 0, 1, 0) == orc.map_one(LAMBDA, 2, n, i, 0)
    for n in (2, 5, 27, 33):
        ex, ey, _ = api.grid_h2d_padded(n).extents
        for y in range(ey):
            for x in range(ex):
                o = api.map_h2d_padded(api.data_coord(x, y, 0), n)
                assert (int(o.is_void), o.target.x, o.target.y, 0, o.level_b, o.index_q) == \
                    orc.map_one(PADDED, 2, n, x, y) or o.is_void and orc.map_one(PADDED, 2, n, x, y)[0] == 1
    for n, T in ((27, 1), (27, 4), (100, 16), (63, 2)):
        for b, t in enumerate(api.decompose_trapezoids(n, T)):
            for y in range(t.ext_y):
                for x in range(t.ext_x):
                    o = api.map_h2d_trapezoid(api.data_coord(x, y, 0), n, T, b)
                    want = orc.map_trapezoid(n, T, b, x, y)
                    got = (int(o.is_void), o.target.x, o.target.y, 0, o.level_b, o.index_q)
                    assert got == want or (o.is_void and want[0] == 1), (n, T, b, x, y)


def test_abi_errors_match_reference():
    for kind, n, T, msg in [(api.map_kind.rb, 0, 1, "grid_rb: n must be >= 1"),
                            (api.map_kind.lambda2d, 0, 1, "grid_lambda: n must be >= 1"),
                            (api.map_kind.h2d_padded, 1, 1, "grid_h2d_padded: n must be >= 2"),
                            (api.map_kind.h2d_trapezoid, 1, 1, "decompose_trapezoids: n must be >= 2"),
                            (api.map_kind.h2d_trapezoid, 10, 0, "decompose_trapezoids: T must be >= 1")]:
        with pytest.raises(api.InvalidArgument, match=msg):
            api.make_grid(kind, 2, n, 1, T)
    with pytest.raises(api.InvalidArgument, match="does not support m=3"):
        api.make_grid(api.map_kind.rb, 3, 8)
    with pytest.raises(api.InvalidArgument, match="map_rb_2d: omega outside the rectangle"):
        api.map_rb_2d(api.data_coord(4, 0, 0), 8)
    with pytest.raises(api.InvalidArgument, match="map_lambda_2d: index out of range"):
        api.map_lambda_2d(15, 5)


def test_trapezoid_union_tiles_every_n(orc):
    # test_maps.cpp:222-234 / acceptance.cpp:108-125: exact cover, <= ceil(log2 n) bands
    for n in range(2, 513):
        for T in (1, 4, 16):
            assert len(orc.decompose_trapezoids(n, T)) <= max(1, (n - 1).bit_length())
            cov, _ = orc.sweep(TRAP, 2, n, 1, T=T)
            assert (cov == 1).all(), (n, T)


def test_restated_edm_and_ca2d_vs_reference_goldens(orc):
    E = G["edm"]
    for row in E["kernel_edm"]:
        if row["side"] <= 255:
            assert orc.state_hash(2, row["side"], orc.kernel_edm(row["side"], row["seed"])) == row["hash"], row
    # every map's launch_edm equals the sequential fill (test_simulator.cpp:199-228)
    seq = {r["side"]: r["hash"] for r in E["kernel_edm"] if r["seed"] == 7}
    for row in E["launch_edm"]:
        side = _side(row["kind"], row["n"], row["rho"])
        want = seq.get(side, orc.state_hash(2, side, orc.kernel_edm(side, 7)))
        assert row["hash"] == want, row
    C2 = G["ca2d"]
    for row in C2["kernel_ca_run"]:
        if row["side"] > 255:
            continue
        st = np.zeros(row["side"] * (row["side"] + 1) // 2, np.uint8)
        init = [r for r in C2["life_init"] if (r["side"], r["seed"]) == (row["side"], row["seed"])]
        st = orc.make_life_state(2, row["side"], row["seed"])
        if init:
            assert orc.state_hash(2, row["side"], st) == init[0]["hash"]
        orc.ca2d_run(row["side"], row["steps"], st)
        assert orc.state_hash(2, row["side"], st) == row["hash"], row
    # 2-D periodic, seed 42, 64 steps
    hashes = {(r["side"], r["steps"], r["seed"]): r["hash"] for r in C2["kernel_ca_run"]}
    assert hashes[(63, 64, 42)] == 8247929562437622423
    assert hashes[(1023, 64, 42)] == 17772433350676739252


def test_edm_points_abi_matches_restated(orc):
    for count, seed in ((14, 7), (1000, 42), (5, 0xC0FFEE)):
        assert (api.make_edm_points(count, seed) == orc.make_edm_points(count, seed)).all()
