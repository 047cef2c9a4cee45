"""Python mirror of the reference's hot-path API (simplexmap, C++ header-only),
backed by the C ABI in libsmx_b200.so. Same names, argument meaning and error
behaviour, so parity tests read like the reference's own tests:

==========================  ==================================================
this module                 reference
==========================  ==================================================
map_kind, grid_spec          maps.hpp:19, :64-92
grid_bb / grid_h2d / grid_h3d  maps.hpp:96-105, :188-198, :285-295
make_grid                    report.hpp:48-66
map_bb / map_h2d / map_h3d   maps.hpp:107-116, :200-207, :302-337
simplex_spec                 core.hpp:28-38
simplex_grid_state           simulator.hpp:37-74 (hash :68-73)
launch_opts / sim_report     simulator.hpp:76-96
launch_map                   simulator.hpp:303-310
launch_accum                 simulator.hpp:313-327
make_life_state              simulator.hpp:390-398
launch_ca                    simulator.hpp:431-463 (dead3d boundary)
verify_exact_cover           simulator.hpp:467-478
==========================  ==================================================

``std::invalid_argument`` surfaces as :class:`InvalidArgument` (a ValueError),
``std::overflow_error`` as :class:`Overflow`. All launches run on the current
CUDA device; there is no CPU execution path.

The ``*_device`` functions are the device-resident entry points (torch CUDA
tensors in, kernels enqueued on the current torch stream, nothing copied).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _lib
from ._lib import EXEC_AUTO, EXEC_BITS, EXEC_BLOCK, EXEC_RUNS, InvalidArgument, Overflow, check, lib


class map_kind(enum.IntEnum):
    bb = 0
    rb = 1
    lambda2d = 2
    h2d = 3
    h2d_trapezoid = 4
    h2d_padded = 5
    h3d = 6


class ca_boundary(enum.IntEnum):
    periodic2d = 0
    dead3d = 1


_KIND_NAMES = {0: "bb", 1: "rb", 2: "lambda", 3: "h2d", 4: "trapezoid", 5: "h2d-padded", 6: "h3d"}


def map_kind_name(k: int) -> str:
    return _KIND_NAMES.get(int(k), "?")


def strict_view(k: int) -> bool:
    """maps.hpp:35-38"""
    return int(k) in (map_kind.h2d, map_kind.h2d_padded, map_kind.h2d_trapezoid, map_kind.h3d)


@dataclass(frozen=True)
class data_coord:
    x: int = 0
    y: int = 0
    z: int = 0


block_coord = data_coord


@dataclass(frozen=True)
class map_outcome:
    is_void: bool
    target: data_coord
    level_b: int
    index_q: int


class grid_spec:
    """grid_spec (maps.hpp:64-92). ``rho`` is assignable, as in the reference."""

    def __init__(self, raw: _lib.smx_grid):
        self._g = raw

    @property
    def kind(self) -> map_kind:
        return map_kind(self._g.kind)

    @property
    def dims(self) -> int:
        return int(self._g.dims)

    @property
    def n(self) -> int:
        return int(self._g.n)

    @property
    def rho(self) -> int:
        return int(self._g.rho)

    @rho.setter
    def rho(self, v: int) -> None:
        self._g.rho = int(v)

    @property
    def threshold(self) -> int:
        return int(self._g.threshold)

    @property
    def extents(self) -> tuple[int, int, int]:
        return tuple(int(v) for v in self._g.extents)

    @property
    def traps(self) -> list[trapezoid_params]:
        """The bands of a trapezoid grid (maps.hpp:259-266), else []."""
        if self.kind != map_kind.h2d_trapezoid:
            return []
        return decompose_trapezoids(self.n, self.threshold)

    def blocks(self) -> int:
        """grid_spec::blocks (maps.hpp:73-82): summed over the bands for trapezoids."""
        return int(lib().smx_grid_blocks(C.byref(self._g)))

    def threads(self) -> int:
        return self.blocks() * self.rho ** self.dims

    def domain_side(self) -> int:
        return self.n - 1 if strict_view(self.kind) else self.n

    def cell_side(self) -> int:
        return self.domain_side() * self.rho

    @property
    def raw(self) -> _lib.smx_grid:
        return self._g

    def __repr__(self) -> str:
        return (f"grid_spec({map_kind_name(self.kind)}, m={self.dims}, n={self.n}, rho={self.rho}, "
                f"extents={self.extents})")


def make_grid(kind: int, m: int, n: int, rho: int = 1, threshold: int = 1) -> grid_spec:
    g = _lib.smx_grid()
    check(lib().smx_make_grid(int(kind), int(m), int(n), int(rho), int(threshold), C.byref(g)))
    return grid_spec(g)


def grid_bb(n: int, m: int) -> grid_spec:
    if m not in (2, 3):
        raise InvalidArgument("grid_bb: m must be 2 or 3")
    return make_grid(map_kind.bb, m, n)


def grid_h2d(n: int) -> grid_spec:
    return make_grid(map_kind.h2d, 2, n)


def grid_h3d(n: int, params=None) -> grid_spec:
    """grid_h3d (maps.hpp:285-295). `params` (analysis.self_similar_params,
    optional): the executable map is the (1/r, beta) = (2, 2) family; any other
    raises InvalidArgument."""
    if params is not None:
        from .analysis import check_executable
        check_executable(params)
    return make_grid(map_kind.h3d, 3, n)


def grid_rb(n: int) -> grid_spec:
    return make_grid(map_kind.rb, 2, n)


def grid_lambda(n: int) -> grid_spec:
    return make_grid(map_kind.lambda2d, 2, n)


def grid_h2d_padded(n: int) -> grid_spec:
    return make_grid(map_kind.h2d_padded, 2, n)


def grid_trapezoids(n: int, T: int) -> grid_spec:
    return make_grid(map_kind.h2d_trapezoid, 2, n, 1, T)


@dataclass(frozen=True)
class trapezoid_params:
    """maps.hpp:49-60"""
    delta_x: int
    delta_y: int
    band: int
    h1: int
    h2: int
    grid_width: int
    valid_side: int
    ext_x: int
    ext_y: int

    def blocks(self) -> int:
        return self.ext_x * self.ext_y


def decompose_trapezoids(n: int, T: int) -> list[trapezoid_params]:
    """maps.hpp:228-257 (the shared arithmetic of include/smx_maps.hpp)."""
    arr = (_lib.smx_trapezoid * 64)()
    cnt = C.c_int32(0)
    check(lib().smx_decompose_trapezoids(int(n), int(T), arr, 64, C.byref(cnt)))
    return [trapezoid_params(*(int(getattr(arr[i], f)) for f, _ in _lib.smx_trapezoid._fields_))
            for i in range(cnt.value)]


def _map_one(kind: int, m: int, n: int, omega) -> map_outcome:
    o = _lib.smx_outcome()
    check(lib().smx_map_one(int(kind), int(m), int(n), int(omega.x), int(omega.y), int(omega.z), C.byref(o)))
    return map_outcome(bool(o.is_void), data_coord(o.x, o.y, o.z), int(o.level_b), int(o.index_q))


def map_bb(omega, n: int, m: int) -> map_outcome:
    return _map_one(map_kind.bb, m, n, omega)


def map_h2d(omega) -> map_outcome:
    return _map_one(map_kind.h2d, 2, 0, omega)


def map_h3d(omega, n: int) -> map_outcome:
    return _map_one(map_kind.h3d, 3, n, omega)


def map_rb_2d(omega, n: int) -> data_coord:
    """maps.hpp:133-141 (returns the data coordinate, as the reference)."""
    return _map_one(map_kind.rb, 2, n, omega).target


def map_lambda_2d(index: int, n: int) -> data_coord:
    """maps.hpp:156-159"""
    return _map_one(map_kind.lambda2d, 2, n, data_coord(int(index), 0, 0)).target


def map_h2d_padded(omega, n: int) -> map_outcome:
    return _map_one(map_kind.h2d_padded, 2, n, omega)


def map_h2d_trapezoid(omega, n: int, T: int, band: int) -> map_outcome:
    """map_h2d_trapezoid (maps.hpp:269-281) on band `band` of decompose_trapezoids(n, T)."""
    o = _lib.smx_outcome()
    check(lib().smx_map_trapezoid(int(n), int(T), int(band), int(omega.x), int(omega.y), C.byref(o)))
    return map_outcome(bool(o.is_void), data_coord(o.x, o.y, o.z), int(o.level_b), int(o.index_q))


def map_outcomes(g: grid_spec) -> np.ndarray:
    """Every block's map_outcome in natural z, y, x order (band after band for
    trapezoid grids) as an (blocks, 8) int32 array {is_void, x, y, z, level_b,
    index_q, 0, 0}, computed on the GPU."""
    out = np.empty((g.blocks(), 8), np.int32)
    check(lib().smx_map_outcomes(C.byref(g.raw), out.ctypes.data, out.shape[0], 0, None))
    return out


def tri_cells(side: int) -> int:
    return side * (side + 1) // 2 if side >= 1 else 0


def tet_cells(side: int) -> int:
    return side * (side + 1) * (side + 2) // 6 if side >= 1 else 0


def tri_linear_index(x: int, y: int) -> int:
    return y * (y + 1) // 2 + x


def tet_layer_prefix(side: int, z: int) -> int:
    return 0 if z == 0 else tet_cells(side) - (0 if z >= side else tet_cells(side - z))


def tet_linear_index(side: int, x: int, y: int, z: int) -> int:
    return tet_layer_prefix(side, z) + tri_linear_index(x, y)


def tri_contains(side: int, x: int, y: int) -> bool:
    return 0 <= x <= y <= side - 1


def tet_contains(side: int, x: int, y: int, z: int) -> bool:
    return 0 <= x <= y and z >= 0 and y <= side - 1 - z


@dataclass
class simplex_spec:
    """core.hpp:28-38"""
    m: int = 2
    n: int = 1

    def __post_init__(self):
        if self.m < 1:
            raise InvalidArgument("simplex_spec: m must be >= 1")
        if self.n < 0:
            raise InvalidArgument("simplex_spec: n must be >= 0")


class simplex_grid_state:
    """Dense packed storage over T(side) / T3(side) (simulator.hpp:37-74).
    ``cells`` is a host numpy array in the reference's packed layout."""

    def __init__(self, m: int, side: int, dtype=np.uint32, cells: np.ndarray | None = None):
        if m not in (2, 3):
            raise InvalidArgument("simplex_grid_state: m must be 2 or 3")
        if side < 1:
            raise InvalidArgument("simplex_grid_state: side must be >= 1")
        self.m, self.side = m, side
        count = tri_cells(side) if m == 2 else tet_cells(side)
        if cells is None:
            cells = np.zeros(count, dtype)
        if cells.shape != (count,):
            raise InvalidArgument("simplex_grid_state: cell array does not match the side")
        self.cells = np.ascontiguousarray(cells)

    def index(self, x: int, y: int, z: int | None = None) -> int:
        if z is None:
            if self.m != 2 or not tri_contains(self.side, x, y):
                raise InvalidArgument("simplex_grid_state: coordinate outside domain")
            return tri_linear_index(x, y)
        if self.m != 3 or not tet_contains(self.side, x, y, z):
            raise InvalidArgument("simplex_grid_state: coordinate outside domain")
        return tet_linear_index(self.side, x, y, z)

    def at(self, x: int, y: int, z: int | None = None):
        return self.cells[self.index(x, y, z)]

    def hash(self) -> int:
        return int(lib().smx_state_hash(self.m, self.side, self.cells.ctypes.data, self.cells.nbytes))


@dataclass
class launch_opts:
    """simulator.hpp:90-96, plus the B200 execution scheme. block_order_salt is
    accepted for API parity; on the GPU the hardware block scheduler decides the
    order and every map here is exact, so results do not depend on it."""
    seed: int = 0
    steps: int = 50
    boundary: ca_boundary = ca_boundary.periodic2d
    record_coverage: bool = True
    block_order_salt: int = 0
    exec: int = EXEC_AUTO
    # B200 extension: launch_ca of a 3-simplex sharded over GPUs of this
    # process (smx_ca_multi): ngpus shards on devices 0..ngpus-1 or `devices`
    ngpus: int = 1
    devices: tuple = ()


@dataclass
class sim_report:
    """simulator.hpp:76-88"""
    m: int = 2
    cell_side: int = 0
    blocks_launched: int = 0
    blocks_void: int = 0
    threads_launched: int = 0
    threads_useful: int = 0
    space_overhead: Fraction = field(default_factory=lambda: Fraction(0))
    coverage: np.ndarray | None = None
    coverage_recorded: bool = True
    state_hash: int = 0
    seed: int = 0


@dataclass
class cover_verdict:
    exact: bool = True
    witness: data_coord = data_coord()
    multiplicity: int = 0


def validate_launch(g: grid_spec, domain: simplex_spec) -> None:
    """simulator.hpp:257-264"""
    if domain.m != g.dims:
        raise InvalidArgument("launch: grid and domain dimensions differ")
    if domain.n != g.domain_side() * g.rho - 1:
        raise InvalidArgument("launch: domain side does not match grid * rho")
    if g.rho < 1:
        raise InvalidArgument("launch: rho must be >= 1")


def _make_report(g: grid_spec, opts: launch_opts) -> sim_report:
    side = g.cell_side()
    rep = sim_report(m=g.dims, cell_side=side, coverage_recorded=opts.record_coverage, seed=opts.seed)
    if opts.record_coverage:
        rep.coverage = np.zeros(tri_cells(side) if g.dims == 2 else tet_cells(side), np.uint32)
    return rep


def _finish(rep: sim_report, cnt: _lib.smx_counters) -> None:
    rep.blocks_launched = int(cnt.blocks_launched)
    rep.blocks_void = int(cnt.blocks_void)
    rep.threads_launched = int(cnt.threads_launched)
    rep.threads_useful = int(cnt.threads_useful)
    if rep.threads_useful > 0:
        rep.space_overhead = Fraction(rep.threads_launched, rep.threads_useful) - 1


def _cov_ptr(rep: sim_report):
    return rep.coverage.ctypes.data if rep.coverage is not None else None


def launch_map(g: grid_spec, domain: simplex_spec, opts: launch_opts | None = None) -> sim_report:
    opts = opts or launch_opts()
    validate_launch(g, domain)
    rep = _make_report(g, opts)
    cnt = _lib.smx_counters()
    ncells = rep.coverage.size if rep.coverage is not None else 0
    check(lib().smx_launch_map(C.byref(g.raw), _cov_ptr(rep), ncells, 0, C.byref(cnt), None))
    _finish(rep, cnt)
    return rep


def launch_accum(g: grid_spec, domain: simplex_spec, state: simplex_grid_state,
                 opts: launch_opts | None = None, stream=None) -> sim_report:
    opts = opts or launch_opts()
    validate_launch(g, domain)
    if state.m != g.dims or state.side != g.cell_side():
        raise InvalidArgument("launch: state does not match the domain")
    if state.cells.dtype != np.uint32:
        raise InvalidArgument("launch_accum: state cells must be u32")
    rep = _make_report(g, opts)
    cnt = _lib.smx_counters()
    check(lib().smx_accum(C.byref(g.raw), state.cells.ctypes.data, state.cells.size, 1, int(opts.exec), 0,
                          _cov_ptr(rep), C.byref(cnt), _raw_stream(stream)))
    _finish(rep, cnt)
    rep.state_hash = state.hash()
    return rep


def kernel_accum(state: simplex_grid_state) -> None:
    """kernel_accum (simulator.hpp:329-331) on the GPU: every cell += 1."""
    if state.cells.dtype != np.uint32:
        raise InvalidArgument("kernel_accum: state cells must be u32")
    check(lib().smx_kernel_accum(state.cells.ctypes.data, state.cells.size, 0, None))


def kernel_edm(points: np.ndarray, state: simplex_grid_state) -> None:
    """kernel_edm (simulator.hpp:377-386) on the GPU."""
    if state.m != 2:
        raise InvalidArgument("kernel_edm: 2-simplex domains only")
    pts = np.ascontiguousarray(points, np.float64)
    if pts.shape[0] != state.side:
        raise InvalidArgument("kernel_edm: need one point per domain side unit")
    check(lib().smx_kernel_edm(pts.ctypes.data, pts.shape[0], state.cells.ctypes.data, state.cells.size, 0, None))


def kernel_ca_run(state: simplex_grid_state, steps: int, boundary: "ca_boundary") -> None:
    """kernel_ca_run (simulator.hpp:402-425) on the GPU, in place."""
    if steps < 0:
        raise InvalidArgument("kernel_ca_run: steps must be >= 0")
    if (boundary == ca_boundary.periodic2d) != (state.m == 2):
        raise InvalidArgument("kernel_ca_run: boundary rule does not fit the domain")
    check(lib().smx_kernel_ca_run(state.m, state.side, state.cells.ctypes.data, state.cells.size, int(steps), 0,
                                  None))


def release_scratch() -> None:
    """Free the calling thread's library scratch on every device (smx_release)."""
    check(lib().smx_release())


def scratch_bytes() -> int:
    """Pooled scratch bytes the calling thread holds (smx_scratch_bytes)."""
    return int(lib().smx_scratch_bytes())


def make_life_state(m: int, side: int, seed: int) -> simplex_grid_state:
    s = simplex_grid_state(m, side, np.uint8)
    check(lib().smx_life_init(m, side, seed, s.cells.ctypes.data, s.cells.size, 0, None))
    return s


def _raw_stream(stream):
    """A cudaStream_t for the C ABI: None (legacy default stream), a raw
    handle (int), or a torch.cuda.Stream."""
    if stream is None:
        return None
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def launch_ca(g: grid_spec, domain: simplex_spec, state: simplex_grid_state,
              opts: launch_opts | None = None, stream=None) -> sim_report:
    """launch_ca (simulator.hpp:431-463) on a host state. `stream` (optional,
    B200 extension): the CUDA stream the call's copies and kernels run on
    (the call still synchronises it before returning)."""
    opts = opts or launch_opts()
    validate_launch(g, domain)
    if state.m != g.dims or state.side != g.cell_side():
        raise InvalidArgument("launch: state does not match the domain")
    if (opts.boundary == ca_boundary.periodic2d) != (g.dims == 2):
        raise InvalidArgument("launch_ca: boundary rule does not fit the domain")
    if opts.steps < 0:
        raise InvalidArgument("launch_ca: steps must be >= 0")
    if state.cells.dtype != np.uint8:
        raise InvalidArgument("launch_ca: state cells must be u8")
    rep = _make_report(g, opts)
    cnt = _lib.smx_counters()
    if g.dims == 3 and (opts.ngpus > 1 or opts.devices):
        if opts.steps > 0:  # step-0 coverage + counters from one map launch
            ncells = rep.coverage.size if rep.coverage is not None else 0
            check(lib().smx_launch_map(C.byref(g.raw), _cov_ptr(rep), ncells, 0, C.byref(cnt), None))
        ca_multi(g, state.cells, int(opts.steps), list(opts.devices) or list(range(opts.ngpus)))
    else:
        check(lib().smx_ca(C.byref(g.raw), state.cells.ctypes.data, state.cells.size, int(opts.steps),
                           int(opts.exec), 0, None, _cov_ptr(rep) if opts.steps > 0 else None,
                           C.byref(cnt) if opts.steps > 0 else None, _raw_stream(stream)))
    if opts.steps > 0:
        _finish(rep, cnt)
    rep.state_hash = state.hash()
    return rep


def make_edm_points(count: int, seed: int) -> np.ndarray:
    """make_edm_points (simulator.hpp:333-343): (count, 2) float64, x then y
    from one seed-keyed splitmix64 stream."""
    out = np.empty((max(count, 0), 2), np.float64)
    check(lib().smx_make_edm_points(int(count), int(seed) & 0xFFFFFFFFFFFFFFFF, out.ctypes.data))
    return out


def launch_edm(g: grid_spec, domain: simplex_spec, points: np.ndarray, state: simplex_grid_state,
               opts: launch_opts | None = None) -> sim_report:
    """launch_edm (simulator.hpp:352-372): cell (x, y) = |p_x - p_y|, f64."""
    opts = opts or launch_opts()
    validate_launch(g, domain)
    if g.dims != 2:
        raise InvalidArgument("launch_edm: 2-simplex domains only")
    if state.m != 2 or state.side != g.cell_side():
        raise InvalidArgument("launch: state does not match the domain")
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    if pts.shape[0] != state.side:
        raise InvalidArgument("launch_edm: need one point per domain side unit")
    if state.cells.dtype != np.float64:
        raise InvalidArgument("launch_edm: state cells must be f64")
    rep = _make_report(g, opts)
    cnt = _lib.smx_counters()
    check(lib().smx_edm(C.byref(g.raw), pts.ctypes.data, pts.shape[0], state.cells.ctypes.data, state.cells.size,
                        int(opts.exec), 0, _cov_ptr(rep), C.byref(cnt), None))
    _finish(rep, cnt)
    rep.state_hash = state.hash()
    return rep


def edm_device(g: grid_spec, points, cells, exec: int = EXEC_AUTO) -> None:
    """Device-resident EDM: points a (side, 2) float64 CUDA tensor, cells f64."""
    check(lib().smx_edm(C.byref(g.raw), _ptr(points), points.shape[0], _ptr(cells), cells.numel(), exec, 1,
                        None, None, _stream()))


def verify_exact_cover(rep: sim_report, domain: simplex_spec) -> cover_verdict:
    """simulator.hpp:467-478: first cell (linear order) whose multiplicity != 1."""
    if domain.m != rep.m or domain.n != rep.cell_side - 1:
        raise InvalidArgument("verify_exact_cover: report/domain mismatch")
    if not rep.coverage_recorded or rep.coverage is None:
        raise InvalidArgument("verify_exact_cover: report has no coverage")
    bad = np.flatnonzero(rep.coverage != 1)
    if bad.size == 0:
        return cover_verdict()
    i = int(bad[0])
    z = 0
    if rep.m == 3:
        while z + 1 < rep.cell_side and tet_layer_prefix(rep.cell_side, z + 1) <= i:
            z += 1
        i -= tet_layer_prefix(rep.cell_side, z)
    y = int((np.sqrt(8.0 * i + 1.0) - 1.0) / 2.0)
    while y > 0 and tri_linear_index(0, y) > i:
        y -= 1
    while tri_linear_index(0, y + 1) <= i:
        y += 1
    return cover_verdict(False, data_coord(i - tri_linear_index(0, y), y, z), int(rep.coverage[bad[0]]))


# ---------------------------------------------------------------------------
# Device-resident entry points (torch CUDA tensors; no copies, current stream).

def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t) -> C.c_void_p:
    if not t.is_cuda:
        raise InvalidArgument("device entry point needs a CUDA tensor")
    if not t.is_contiguous():
        raise InvalidArgument("device entry point needs a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def accum_device(g: grid_spec, cells, passes: int = 1, exec: int = EXEC_RUNS) -> None:
    check(lib().smx_accum(C.byref(g.raw), _ptr(cells), cells.numel(), passes, exec, 1, None, None, _stream()))


def accum_range_device(g: grid_spec, cells, passes: int, wy_lo: int, wy_hi: int,
                       exec: int = EXEC_RUNS, counters: bool = True) -> dict | None:
    """ACCUM over grid rows [wy_lo, wy_hi) only (a multi-GPU shard);
    returns that range's launch counters (counters=False: none, no sync)."""
    cnt = _lib.smx_counters()
    check(lib().smx_accum_range(C.byref(g.raw), _ptr(cells), cells.numel(), passes, exec, wy_lo, wy_hi,
                                C.byref(cnt) if counters else None, _stream()))
    if not counters:
        return None
    return {"blocks_launched": int(cnt.blocks_launched), "blocks_void": int(cnt.blocks_void),
            "threads_launched": int(cnt.threads_launched), "threads_useful": int(cnt.threads_useful)}


def life_init_device(m: int, side: int, seed: int, cells) -> None:
    check(lib().smx_life_init(m, side, seed, _ptr(cells), cells.numel(), 1, _stream()))


def ca_step_device(g: grid_spec, cur, nxt, exec: int = EXEC_AUTO) -> None:
    check(lib().smx_ca_step(C.byref(g.raw), _ptr(cur), _ptr(nxt), cur.numel(), exec, _stream()))


def ca_step_range_device(g: grid_spec, cur, nxt, wz_lo: int, wz_hi: int, exec: int = EXEC_AUTO) -> None:
    check(lib().smx_ca_step_range(C.byref(g.raw), _ptr(cur), _ptr(nxt), cur.numel(), wz_lo, wz_hi, exec,
                                  _stream()))


def ca_device(g: grid_spec, cells, steps: int, exec: int = EXEC_AUTO, scratch=None) -> None:
    check(lib().smx_ca(C.byref(g.raw), _ptr(cells), cells.numel(), steps, exec, 1,
                       _ptr(scratch) if scratch is not None else None, None, None, _stream()))


def ca_multi(g: grid_spec, cells, steps: int, devices) -> None:
    """launch_ca over several GPUs of this process (smx_ca_multi): `cells` a
    host numpy u8 state or a CUDA tensor on devices[0]; `devices` ordinals
    (may repeat: shards on one device)."""
    devs = (C.c_int32 * len(devices))(*devices)
    if isinstance(cells, np.ndarray):
        check(lib().smx_ca_multi(C.byref(g.raw), cells.ctypes.data, cells.size, int(steps), devs, len(devices), 0,
                                 None, None))
    else:
        check(lib().smx_ca_multi(C.byref(g.raw), _ptr(cells), cells.numel(), int(steps), devs, len(devices), 1,
                                 None, _stream()))


def map_kernel_device(g: grid_spec) -> None:
    check(lib().smx_map_kernel(C.byref(g.raw), _stream()))


def launch_map_device(g: grid_spec, coverage=None) -> sim_report:
    cnt = _lib.smx_counters()
    check(lib().smx_launch_map(C.byref(g.raw), _ptr(coverage) if coverage is not None else None,
                               coverage.numel() if coverage is not None else 0, 1, C.byref(cnt), _stream()))
    rep = sim_report(m=g.dims, cell_side=g.cell_side(), coverage_recorded=coverage is not None)
    _finish(rep, cnt)
    return rep


def tiles_pack_device(g: grid_spec, cells, tiles, out) -> None:
    check(lib().smx_tiles_pack(C.byref(g.raw), _ptr(cells), _ptr(tiles), tiles.shape[0], _ptr(out), _stream()))


def tiles_unpack_device(g: grid_spec, cells, tiles, buf) -> None:
    check(lib().smx_tiles_unpack(C.byref(g.raw), _ptr(cells), _ptr(tiles), tiles.shape[0], _ptr(buf), _stream()))


def bits_tiles_pack_device(g: grid_spec, bits, tiles, out) -> None:
    check(lib().smx_bits_tiles_pack(C.byref(g.raw), _ptr(bits), _ptr(tiles), tiles.shape[0], _ptr(out), _stream()))


def bits_tiles_unpack_device(g: grid_spec, bits, tiles, buf) -> None:
    check(lib().smx_bits_tiles_unpack(C.byref(g.raw), _ptr(bits), _ptr(tiles), tiles.shape[0], _ptr(buf),
                                      _stream()))


def bits_tile_bytes(g: grid_spec) -> int:
    return int(lib().smx_bits_tile_bytes(C.byref(g.raw), 1))


def bits_buffer(g: grid_spec):
    """A device bit shadow for the x-run engine stages (with TMA-read slack)."""
    import torch
    n = int(lib().smx_bits_bytes(C.byref(g.raw)))
    if n == 0:
        raise InvalidArgument("bits_buffer: 3-simplex grids only")
    return torch.zeros((n + 511) // 4, dtype=torch.int32, device="cuda")


def bits_pack_device(g: grid_spec, cells, bits) -> None:
    check(lib().smx_bits_pack(C.byref(g.raw), _ptr(cells), cells.numel(), _ptr(bits), _stream()))


def bits_step_device(g: grid_spec, bits_in, bits_out, wz_lo: int = 0, wz_hi: int | None = None) -> None:
    hi = g.extents[2] if wz_hi is None else wz_hi
    check(lib().smx_bits_step(C.byref(g.raw), _ptr(bits_in), _ptr(bits_out), wz_lo, hi, _stream()))


def bits_run_device(g: grid_spec, bits_a, bits_b, steps: int) -> None:
    """The engine stage: map once + one persistent launch of `steps` steps
    (result in bits_a for even steps, bits_b for odd)."""
    check(lib().smx_bits_run(C.byref(g.raw), _ptr(bits_a), _ptr(bits_b), steps, _stream()))


def ca_engine(g: grid_spec) -> str:
    """The multi-step CA engine smx_ca uses for this grid: "chunk" or "column"."""
    return {0: "chunk", 1: "column"}.get(int(lib().smx_ca_engine(C.byref(g.raw))), "none")


def bits_plan_capacity(g: grid_spec) -> int:
    return int(lib().smx_bits_plan_capacity(C.byref(g.raw)))


def bits_plan_device(g: grid_spec, wz_lo: int, wz_hi: int):
    """The engine's plan for the blocks with wz in [wz_lo, wz_hi): returns
    (chunks, count) device tensors — chunks (capacity, 4) int32 rows
    {x0, y0, z0, owned width} in cells, count (1,) int32 = chunks used."""
    import torch
    cap = max(bits_plan_capacity(g), 1)
    chunks = torch.empty((cap, 4), dtype=torch.int32, device="cuda")
    count = torch.zeros(1, dtype=torch.int32, device="cuda")
    check(lib().smx_bits_plan(C.byref(g.raw), wz_lo, wz_hi, _ptr(chunks), _ptr(count), _stream()))
    return chunks, count


def bits_run_list_device(g: grid_spec, bits_in, bits_out, chunks, count) -> None:
    """One Life step bits_in -> bits_out over an explicit chunk list."""
    check(lib().smx_bits_run_list(C.byref(g.raw), _ptr(bits_in), _ptr(bits_out), _ptr(chunks), _ptr(count),
                                  _stream()))


def bits_unpack_device(g: grid_spec, bits, cells) -> None:
    check(lib().smx_bits_unpack(C.byref(g.raw), _ptr(bits), _ptr(cells), cells.numel(), _stream()))


def state_hash(m: int, side: int, arr: np.ndarray) -> int:
    a = np.ascontiguousarray(arr)
    return int(lib().smx_state_hash(m, side, a.ctypes.data, a.nbytes))


__all__ = [n for n in dir() if not n.startswith("_")] + ["EXEC_AUTO", "EXEC_BLOCK", "EXEC_RUNS"]
