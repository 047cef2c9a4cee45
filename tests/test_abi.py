"""The C ABI boundary without a GPU (CPU suite): the library loads, exports every
symbol include/smx_b200.h declares, and its host-side pieces — make_grid
validation, the shared map arithmetic (include/smx_maps.hpp compiled for the
host), the state hash — agree with the oracle and the reference's contracts."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden
from oracle.oracle import BB, H2D, H3D
from paper_2208_11617_b200 import _lib, api


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "smx_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\*?\s+\**(smx_\w+)\(", text, re.M)))


def test_header_symbols_exported():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.exported_symbols())


def test_struct_layouts_match_header():
    assert C.sizeof(_lib.smx_outcome) == 32
    assert C.sizeof(_lib.smx_counters) == 32
    assert C.sizeof(_lib.smx_grid) == 56


def test_grid_shapes():
    # test_maps.cpp:113-118, :237-238
    assert api.grid_h2d(8).extents == (4, 7, 1)
    assert api.grid_h2d(8).blocks() == 28
    assert api.grid_h2d(2).extents == (1, 1, 1)
    assert api.grid_h2d(1024).blocks() == 523776
    assert api.grid_h3d(4).extents == (2, 2, 3)
    assert api.grid_h3d(64).blocks() == 49152
    assert api.grid_bb(8, 3).blocks() == 512
    assert api.grid_bb(1, 2).blocks() == 1
    g = api.make_grid(api.map_kind.h3d, 3, 256, 8)
    assert (g.rho, g.cell_side(), g.domain_side()) == (8, 2040, 255)


@pytest.mark.parametrize("call,msg", [
    (lambda: api.grid_h2d(9), "grid_h2d: n must be a power of two >= 2"),
    (lambda: api.grid_h2d(1), "grid_h2d: n must be a power of two >= 2"),
    (lambda: api.grid_h3d(2), "grid_h3d: n must be a power of two >= 4"),
    (lambda: api.grid_h3d(24), "grid_h3d: n must be a power of two >= 4"),
    (lambda: api.grid_bb(0, 2), "grid_bb: n must be >= 1"),
    (lambda: api.grid_bb(4, 4), "grid_bb: m must be 2 or 3"),
    (lambda: api.make_grid(api.map_kind.h3d, 2, 8), "map h3d does not support m=2"),
    (lambda: api.make_grid(api.map_kind.h2d, 2, 8, 0), "rho must be >= 1"),
    (lambda: api.map_bb(api.block_coord(8, 0, 0), 8, 2), "map_bb: omega outside the n^m grid"),
    (lambda: api.map_bb(api.block_coord(0, 0, 0), 8, 4), "map_bb: m must be 2 or 3"),
    (lambda: api.map_h3d(api.block_coord(0, 0, 99), 8), "map_h3d: omega outside the grid"),
    (lambda: api.map_h2d(api.block_coord(-1, 0, 0)), "map_h2d: omega components must be >= 0"),
])
def test_contract_violations_raise_invalid_argument(call, msg):
    with pytest.raises(api.InvalidArgument, match=re.escape(msg)):
        call()


def test_host_maps_equal_oracle(orc):
    for kind, m, n in [(H2D, 2, 2), (H2D, 2, 64), (H3D, 3, 4), (H3D, 3, 32), (BB, 2, 9), (BB, 3, 7)]:
        want = orc.map_outcomes(kind, m, n)
        ex, ey, ez = orc.grid(kind, m, n)
        i = 0
        for z in range(ez):
            for y in range(ey):
                for x in range(ex):
                    w = api.block_coord(x, y, z)
                    o = (api.map_h2d(w) if kind == H2D else api.map_h3d(w, n) if kind == H3D
                         else api.map_bb(w, n, m))
                    got = (int(o.is_void), o.target.x, o.target.y, o.target.z, o.level_b, o.index_q)
                    assert got == tuple(int(v) for v in want[i]), (kind, n, x, y, z)
                    i += 1


def test_pinned_points():
    assert api.map_h2d(api.block_coord(3, 0, 0)).target == api.data_coord(6, 7, 0)
    o = api.map_h2d(api.block_coord(2, 1, 0))
    assert (o.target, o.level_b, o.index_q) == (api.data_coord(4, 6, 0), 2, 1)
    assert api.map_h3d(api.block_coord(0, 0, 0), 8).target == api.data_coord(0, 5, 0)
    assert api.map_bb(api.block_coord(7, 2, 0), 8, 2).is_void


def test_state_hash_equals_oracle(orc):
    rng = np.random.default_rng(3)
    for m, side in [(2, 17), (3, 9)]:
        a = rng.integers(0, 2, api.tri_cells(side) if m == 2 else api.tet_cells(side)).astype(np.uint8)
        assert api.state_hash(m, side, a) == orc.state_hash(m, side, a)
    st = api.simplex_grid_state(2, 1023)
    st.cells[:] = 1
    want = {(r["kind"], r["n"], r["rho"]): r["hash"] for r in golden("accum.json")["launch_accum"]}
    assert st.hash() == want[(H2D, 1024, 1)]


def test_state_accessors_reject_outside():
    # test_simulator.cpp:380-391
    s = api.simplex_grid_state(2, 8)
    with pytest.raises(api.InvalidArgument):
        s.at(5, 3)
    with pytest.raises(api.InvalidArgument):
        s.at(0, 8)
    t = api.simplex_grid_state(3, 8)
    with pytest.raises(api.InvalidArgument):
        t.at(0, 4, 4)
    assert t.index(0, 4, 3) == api.tet_linear_index(8, 0, 4, 3)


def test_launch_validation_before_any_device_work():
    g = api.grid_h2d(16)
    with pytest.raises(api.InvalidArgument, match="domain side does not match"):
        api.launch_map(g, api.simplex_spec(2, 15))
    with pytest.raises(api.InvalidArgument, match="dimensions differ"):
        api.launch_map(g, api.simplex_spec(3, 14))
    with pytest.raises(api.InvalidArgument, match="state does not match"):
        api.launch_accum(g, api.simplex_spec(2, 14), api.simplex_grid_state(2, 16))
    life = api.simplex_grid_state(2, 15, np.uint8)
    with pytest.raises(api.InvalidArgument, match="boundary rule"):
        api.launch_ca(g, api.simplex_spec(2, 14), life,
                      api.launch_opts(boundary=api.ca_boundary.dead3d))


def test_library_has_sm100a_code():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_missing_library_fails_loudly(monkeypatch):
    """No CPU fallback: without the sm_100a library every entry point raises."""
    from paper_2208_11617_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libsmx_b200.so")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.lib()


def test_accum_range_contract_checked_before_device_work():
    """smx_accum_range shards 2-D non-trapezoid grids by rows; other grids are
    rejected with the contract message before any CUDA call."""
    L = _lib.lib()
    for g in (api.grid_h3d(8), api.grid_trapezoids(9, 1)):
        rc = L.smx_accum_range(C.byref(g.raw), None, 0, 1, api.EXEC_RUNS, 0, 1, None, None)
        assert rc == 1 and b"row ranges" in L.smx_last_error()


def test_engine_choice_and_rho16_rules_host_side():
    """smx_ca_engine (host-side decision, no device work): the column engine
    for states >= 96 M cells, the chunk engine below; none for 2-D grids."""
    big = api.make_grid(api.map_kind.h3d, 3, 256, 8)     # C5: 1.42 G cells
    c4 = api.make_grid(api.map_kind.h3d, 3, 128, 8)      # C4: 175 M
    c2 = api.make_grid(api.map_kind.h3d, 3, 64, 4)       # C2: 2.7 M
    assert api.ca_engine(big) == "column" and api.ca_engine(c4) == "column"
    assert api.ca_engine(c2) == "chunk"
    assert api.ca_engine(api.make_grid(api.map_kind.h3d, 3, 128, 16)) == "column"
    assert api.ca_engine(api.grid_h2d(64)) == "none"
