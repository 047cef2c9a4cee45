"""Verification sweeps and CSV report emission on the GPU.

Mirror of the reference's report layer (report.hpp): the same rows, the same
column order and schema tags (``slx-1`` / ``slx-an-1`` / ``slx-sim-1``), the
same round-half-up decimals, so identical inputs give byte-identical text —
but every grid of a sweep is one ``launch_map`` on the B200 with the coverage
multiset kept on the device and the exact-cover verdict reduced there
(``smx_verify_cover``). The reference's trapezoid sweep over n in [2, 4096]
x T in {1, 4, 16} (acceptance.cpp:108-125) takes minutes on the CPU and
seconds here.

    measure_grid       report.hpp:190-203   (one launch, optional cover check)
    verify_sweep       report.hpp:324-332   (cover-checking sweep; multiplicity capped at 255
                                             like measure_grid_compact, :287-321)
    analyze_sweep      report.hpp:335-342   (count-only)
    parse_n_range / expand_n_range          report.hpp:73-110
    scheme_overhead_limit                   report.hpp:345-352
    csv_measure / csv_analyze / csv_simulate  report.hpp:386-446
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from fractions import Fraction

from . import _lib, api
from ._lib import check, lib

CSV_SCHEMA_MEASURE = "slx-1"
CSV_SCHEMA_SIMULATE = "slx-sim-1"
CSV_SCHEMA_ANALYZE = "slx-an-1"
CSV_MEASURE_COLUMNS = ("map,m,n,rho,blocks_launched,blocks_void,threads_launched,threads_useful,"
                       "overhead_num,overhead_den,overhead_decimal")


@dataclass
class measure_row:
    """report.hpp:158-171"""
    kind: int = api.map_kind.bb
    m: int = 2
    n: int = 1
    rho: int = 1
    blocks_launched: int = 0
    blocks_void: int = 0
    threads_launched: int = 0
    threads_useful: int = 0
    overhead: Fraction = field(default_factory=lambda: Fraction(0))
    exact: bool = False
    witness: api.data_coord = api.data_coord()
    multiplicity: int = 0


@dataclass(frozen=True)
class n_range:
    lo: int = 1
    hi: int = 1
    pow2_only: bool = False


def parse_n_range(text: str) -> n_range:
    """report.hpp:73-96: "N", "LO..HI", "LO..HI(pow2)"."""
    def parse_int(s: str) -> int:
        if not s or not s.isdigit():
            raise api.InvalidArgument("bad n-range literal: " + s)
        return int(s)

    if ".." not in text:
        v = parse_int(text)
        return n_range(v, v, False)
    lo_s, rest = text.split("..", 1)
    lo = parse_int(lo_s)
    pow2 = len(rest) > 6 and rest.endswith("(pow2)")
    if pow2:
        rest = rest[:-6]
    hi = parse_int(rest)
    if lo < 1 or hi < lo:
        raise api.InvalidArgument("bad n-range: " + text)
    return n_range(lo, hi, pow2)


def expand_n_range(r: n_range) -> list[int]:
    """report.hpp:98-110"""
    if not r.pow2_only:
        return list(range(r.lo, r.hi + 1))
    out, n = [], 1
    while n <= r.hi:
        if n >= r.lo:
            out.append(n)
        if n > r.hi // 2:
            break
        n *= 2
    return out


def _coord_at(m: int, side: int, index: int) -> api.data_coord:
    """tri_coord_at / tet_coord_at (core.hpp:151-164)"""
    def tri(i: int):
        y = int(((8 * i + 1) ** 0.5 - 1) / 2)
        while y > 0 and y * (y + 1) // 2 > i:
            y -= 1
        while (y + 1) * (y + 2) // 2 <= i:
            y += 1
        return i - y * (y + 1) // 2, y
    if m == 2:
        x, y = tri(index)
        return api.data_coord(x, y, 0)
    z = 0
    while z + 1 < side and api.tet_layer_prefix(side, z + 1) <= index:
        z += 1
    x, y = tri(index - api.tet_layer_prefix(side, z))
    return api.data_coord(x, y, z)


def _row(g: api.grid_spec, rep: api.sim_report) -> measure_row:
    """row_from_report (report.hpp:173-186)"""
    return measure_row(g.kind, g.dims, g.n, g.rho, rep.blocks_launched, rep.blocks_void, rep.threads_launched,
                       rep.threads_useful, rep.space_overhead)


def measure_grid(g: api.grid_spec, check_cover: bool = True, _cap: int | None = None) -> measure_row:
    """report.hpp:190-203: one launch of the map kernel on the GPU into a
    device-resident coverage multiset, the cover verdict reduced there
    (smx_measure_grid); only the counters and the verdict reach the host."""
    side = g.cell_side()
    cells = api.tri_cells(side) if g.dims == 2 else api.tet_cells(side)
    cnt = _lib.smx_counters()
    first = C.c_uint64(cells)
    mult = C.c_uint32(0)
    check(lib().smx_measure_grid(C.byref(g.raw), 1 if check_cover else 0, C.byref(cnt), C.byref(first),
                                 C.byref(mult), api._stream()))
    rep = api.sim_report(m=g.dims, cell_side=side)
    api._finish(rep, cnt)
    row = _row(g, rep)
    if check_cover:
        row.exact = first.value == cells
        if not row.exact:
            row.witness = _coord_at(g.dims, side, int(first.value))
            row.multiplicity = int(mult.value) if _cap is None else min(int(mult.value), _cap)
    return row


def verify_sweep(kind: int, m: int, ns: list[int], rho: int = 1, threshold: int = 1) -> list[measure_row]:
    """report.hpp:324-332 (rows in input order; multiplicity capped at 255 as
    measure_grid_compact's byte marks do)."""
    return [measure_grid(api.make_grid(kind, m, n, rho, threshold), True, _cap=255) for n in ns]


def analyze_sweep(kind: int, m: int, ns: list[int], rho: int = 1, threshold: int = 1) -> list[measure_row]:
    """report.hpp:335-342: count-only."""
    return [measure_grid(api.make_grid(kind, m, n, rho, threshold), False) for n in ns]


def scheme_overhead_limit(kind: int, m: int) -> Fraction:
    """report.hpp:345-352; bb_waste_fraction(m) = m! - 1 (core.hpp:125-128)."""
    if kind == api.map_kind.bb:
        f = 1
        for i in range(2, m + 1):
            f *= i
        return Fraction(f - 1)
    if kind == api.map_kind.h2d_padded:
        return Fraction(3)
    if kind == api.map_kind.h3d:
        return Fraction(1, 8)
    return Fraction(0)


def decimal_string(r: Fraction, digits: int = 9) -> str:
    """rational::to_decimal_string (rational.hpp:129-144): fixed point,
    round half up on the magnitude."""
    n = abs(r.numerator)
    scale = 10 ** digits
    scaled = n * scale
    q, rem = divmod(scaled, r.denominator)
    if rem * 2 >= r.denominator:
        q += 1
    s = "-" if (r < 0 and q != 0) else ""
    s += str(q // scale)
    if digits > 0:
        s += "." + str(q % scale).zfill(digits)
    return s


def _rational_fields(r: Fraction) -> str:
    return f"{r.numerator},{r.denominator},{decimal_string(r)}"


def _measure_fields(r: measure_row) -> str:
    return (f"{api.map_kind_name(r.kind)},{r.m},{r.n},{r.rho},{r.blocks_launched},{r.blocks_void},"
            f"{r.threads_launched},{r.threads_useful},{_rational_fields(r.overhead)}")


def csv_measure(rows: list[measure_row]) -> str:
    """report.hpp:386-398"""
    out = "schema," + CSV_MEASURE_COLUMNS + "\n"
    for r in rows:
        out += CSV_SCHEMA_MEASURE + "," + _measure_fields(r) + "\n"
    return out


def csv_analyze(rows: list[measure_row]) -> str:
    """report.hpp:400-412"""
    out = "schema," + CSV_MEASURE_COLUMNS + ",limit_num,limit_den,limit_decimal\n"
    for r in rows:
        out += (CSV_SCHEMA_ANALYZE + "," + _measure_fields(r) + "," + _rational_fields(
            scheme_overhead_limit(r.kind, r.m)) + "\n")
    return out


@dataclass
class simulate_row:
    """report.hpp:414-420"""
    base: measure_row
    kernel: str = "map"  # kernel_kind_name: map, accum, edm, ca
    steps: int = 0
    seed: int = 0
    state_hash: int = 0


def csv_simulate(rows: list[simulate_row]) -> str:
    """report.hpp:422-446"""
    out = "schema," + CSV_MEASURE_COLUMNS + ",kernel,steps,seed,state_hash\n"
    for r in rows:
        out += (CSV_SCHEMA_SIMULATE + "," + _measure_fields(r.base) + f",{r.kernel},{r.steps},{r.seed},"
                f"{r.state_hash}\n")
    return out


def text_report(rows: list[measure_row], verified: bool) -> str:
    """report.hpp:483-511: one human-readable line per row."""
    out = ""
    for r in rows:
        ov = Fraction(r.overhead)
        frac = str(ov.numerator) if ov.denominator == 1 else f"{ov.numerator}/{ov.denominator}"
        out += (f"map={api.map_kind_name(r.kind)} m={r.m} n={r.n} rho={r.rho} blocks={r.blocks_launched} "
                f"void={r.blocks_void} threads={r.threads_launched} useful={r.threads_useful} "
                f"overhead={frac} ({decimal_string(ov, 6)})")
        if verified:
            out += " Exact" if r.exact else f" NotExact witness={witness_text(r)} mult={r.multiplicity}"
        out += "\n"
    return out


def witness_text(r: measure_row) -> str:
    """report.hpp:475-480"""
    out = f"({r.witness.x},{r.witness.y}"
    if r.m == 3:
        out += f",{r.witness.z}"
    return out + ")"


__all__ = ["measure_row", "n_range", "parse_n_range", "expand_n_range", "measure_grid", "verify_sweep",
           "analyze_sweep", "scheme_overhead_limit", "decimal_string", "csv_measure", "csv_analyze",
           "simulate_row", "csv_simulate", "witness_text", "text_report", "CSV_SCHEMA_MEASURE", "CSV_SCHEMA_SIMULATE",
           "CSV_SCHEMA_ANALYZE", "CSV_MEASURE_COLUMNS", "_lib"]
