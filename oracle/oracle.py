"""TEST INFRASTRUCTURE ONLY — ctypes loaders for the two CPU checkers.

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this module. The product package
``paper_2208_11617_b200`` never imports it.

* ``Restated``  — oracle/libsmx_oracle.so, the plain-C restatement (smx_oracle.c).
* ``Reference`` — oracle/_ref/libsmx_ref.so, the unmodified reference headers
  compiled in place (ref_harness.cpp); absent if it was never built.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATED_SO = os.path.join(HERE, "libsmx_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsmx_ref.so")

# map_kind ordinals (maps.hpp:19)
BB, RB, LAMBDA, H2D, TRAP, PADDED, H3D = range(7)

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def tri_cells(side: int) -> int:
    return side * (side + 1) // 2 if side >= 1 else 0


def tet_cells(side: int) -> int:
    return side * (side + 1) * (side + 2) // 6 if side >= 1 else 0


def cells_of(m: int, side: int) -> int:
    return tri_cells(side) if m == 2 else tet_cells(side)


def ncpu() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class OracleError(RuntimeError):
    pass


class Restated:
    """The plain-C restatement (oracle/smx_oracle.c)."""

    def __init__(self, path: str = RESTATED_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_grid.argtypes = [C.c_int, C.c_int, C.c_int64, _i64p]
        L.orc_map_outcomes.argtypes = [C.c_int, C.c_int, C.c_int64, _i64p, C.c_uint64]
        L.orc_map_h2d.argtypes = [C.c_int64, C.c_int64, _i64p]
        L.orc_map_h3d.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, _i64p]
        L.orc_map_bb.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int, _i64p]
        L.orc_sweep.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, _u64p]
        L.orc_state_hash.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_uint64]
        L.orc_state_hash.restype = C.c_uint64
        L.orc_make_life_state.argtypes = [C.c_int, C.c_int64, C.c_uint64, _u8p, C.c_uint64, C.c_int]
        L.orc_ca3d_run.argtypes = [C.c_int64, C.c_int64, _u8p, C.c_uint64, C.c_int]
        L.orc_ca3d_run_literal.argtypes = [C.c_int64, C.c_int64, _u8p, C.c_uint64]
        L.orc_first_defect.argtypes = [C.c_int, C.c_int64, _u32p, C.c_uint64, _i64p, _u64p]
        L.orc_tet_layer_prefix.argtypes = [C.c_int64, C.c_int64]
        L.orc_tet_layer_prefix.restype = C.c_uint64
        L.orc_grid_blocks.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64]
        L.orc_grid_blocks.restype = C.c_uint64
        L.orc_map_outcomes_t.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, _i64p, C.c_uint64]
        L.orc_sweep_t.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                  _u64p]
        L.orc_decompose_trapezoids.argtypes = [C.c_int64, C.c_int64, _i64p, C.c_int, C.POINTER(C.c_int)]
        L.orc_map_trapezoid.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_int64, C.c_int64, _i64p]
        L.orc_map_rb.argtypes = [C.c_int64, C.c_int64, C.c_int64, _i64p]
        L.orc_map_lambda.argtypes = [C.c_uint64, C.c_int64, _i64p]
        L.orc_map_padded.argtypes = [C.c_int64, C.c_int64, C.c_int64, _i64p]
        L.orc_make_edm_points.argtypes = [C.c_int64, C.c_uint64, _f64p]
        L.orc_kernel_edm.argtypes = [C.c_int64, _f64p, _f64p]
        L.orc_ca2d_run.argtypes = [C.c_int64, C.c_int64, _u8p, C.c_uint64]
        self.L = L

    @staticmethod
    def _ok(rc: int, what: str) -> None:
        if rc != 0:
            raise OracleError(f"{what}: status {rc}")

    def grid(self, kind: int, m: int, n: int):
        e = np.zeros(3, np.int64)
        self._ok(self.L.orc_grid(kind, m, n, e), "grid")
        return tuple(int(v) for v in e)

    def blocks(self, kind: int, m: int, n: int, T: int = 1) -> int:
        return int(self.L.orc_grid_blocks(kind, m, n, T))

    def map_outcomes(self, kind: int, m: int, n: int, T: int = 1) -> np.ndarray:
        nb = self.blocks(kind, m, n, T)
        if nb == 0:
            raise OracleError("map_outcomes: invalid grid")
        out = np.zeros((nb, 6), np.int64)
        self._ok(self.L.orc_map_outcomes_t(kind, m, n, T, out, nb), "map_outcomes")
        return out

    def map_one(self, kind: int, m: int, n: int, x: int, y: int, z: int = 0):
        o = np.zeros(6, np.int64)
        if kind == H2D:
            rc = self.L.orc_map_h2d(x, y, o)
        elif kind == H3D:
            rc = self.L.orc_map_h3d(x, y, z, n, o)
        elif kind == RB:
            rc = self.L.orc_map_rb(x, y, n, o)
        elif kind == LAMBDA:
            rc = self.L.orc_map_lambda(x, n, o)
        elif kind == PADDED:
            rc = self.L.orc_map_padded(x, y, n, o)
        else:
            rc = self.L.orc_map_bb(x, y, z, n, m, o)
        self._ok(rc, "map_one")
        return tuple(int(v) for v in o)

    def make_edm_points(self, count: int, seed: int) -> np.ndarray:
        out = np.zeros((count, 2), np.float64)
        self.L.orc_make_edm_points(count, seed, out)
        return out

    def kernel_edm(self, side: int, seed: int) -> np.ndarray:
        pts = self.make_edm_points(side, seed)
        cells = np.zeros(tri_cells(side), np.float64)
        self.L.orc_kernel_edm(side, pts, cells)
        return cells

    def ca2d_run(self, side: int, steps: int, cells: np.ndarray) -> np.ndarray:
        self._ok(self.L.orc_ca2d_run(side, steps, cells, cells.size), "ca2d_run")
        return cells

    def decompose_trapezoids(self, n: int, T: int) -> list[dict]:
        out = np.zeros(9 * 64, np.int64)
        c = C.c_int(0)
        self._ok(self.L.orc_decompose_trapezoids(n, T, out, 64, C.byref(c)), "decompose_trapezoids")
        keys = ("delta_x", "delta_y", "band", "h1", "h2", "grid_width", "valid_side", "ext_x", "ext_y")
        return [dict(zip(keys, (int(v) for v in out[9 * i:9 * i + 9]))) for i in range(c.value)]

    def map_trapezoid(self, n: int, T: int, band: int, x: int, y: int):
        o = np.zeros(6, np.int64)
        self._ok(self.L.orc_map_trapezoid(n, T, band, x, y, o), "map_trapezoid")
        return tuple(int(v) for v in o)

    def sweep(self, kind: int, m: int, n: int, rho: int, coverage: bool = True,
              cells: np.ndarray | None = None, T: int = 1):
        strict = kind in (H2D, TRAP, PADDED, H3D)
        side = (n - 1 if strict else n) * rho
        cov = np.zeros(cells_of(m, side), np.uint32) if coverage else None
        cnt = np.zeros(4, np.uint64)
        self._ok(self.L.orc_sweep_t(kind, m, n, rho, T,
                                    cov.ctypes.data if cov is not None else None,
                                    cells.ctypes.data if cells is not None else None, cnt), "sweep")
        return cov, [int(v) for v in cnt]

    def state_hash(self, m: int, side: int, arr: np.ndarray) -> int:
        a = np.ascontiguousarray(arr)
        return int(self.L.orc_state_hash(m, side, a.ctypes.data, a.nbytes))

    def make_life_state(self, m: int, side: int, seed: int, threads: int | None = None) -> np.ndarray:
        out = np.empty(cells_of(m, side), np.uint8)
        self._ok(self.L.orc_make_life_state(m, side, seed, out, out.size, threads or ncpu()), "life")
        return out

    def ca3d_run(self, side: int, steps: int, cells: np.ndarray, threads: int | None = None) -> np.ndarray:
        self._ok(self.L.orc_ca3d_run(side, steps, cells, cells.size, threads or ncpu()), "ca3d")
        return cells

    def ca3d_run_literal(self, side: int, steps: int, cells: np.ndarray) -> np.ndarray:
        self._ok(self.L.orc_ca3d_run_literal(side, steps, cells, cells.size), "ca3d_literal")
        return cells

    def first_defect(self, m: int, side: int, cov: np.ndarray):
        w = np.zeros(3, np.int64)
        mult = np.zeros(1, np.uint64)
        exact = self.L.orc_first_defect(m, side, cov, cov.size, w, mult)
        return bool(exact), tuple(int(v) for v in w), int(mult[0])


class Reference:
    """The unmodified reference headers compiled in place (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_make_grid.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, _i64p,
                                    _u64p, _i64p]
        L.ref_map_outcomes.argtypes = [C.c_int, C.c_int, C.c_int64, _i64p, C.c_uint64]
        L.ref_map_one.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _i64p]
        L.ref_launch_map.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                     C.c_uint64, C.c_uint64, _u64p]
        L.ref_launch_accum.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                       _u32p, C.c_uint64, _u64p, _u64p, C.POINTER(C.c_double)]
        L.ref_make_life_state.argtypes = [C.c_int, C.c_int64, C.c_uint64, _u8p, C.c_uint64]
        L.ref_accum_sample.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                       C.c_int, _f64p, _u64p]
        L.ref_kernel_ca_run.argtypes = [C.c_int, C.c_int64, C.c_int64, _u8p, C.c_uint64,
                                        C.POINTER(C.c_double)]
        L.ref_launch_ca.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                    _u8p, C.c_uint64, _u64p, _u64p, C.POINTER(C.c_double)]
        L.ref_state_hash.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_uint64]
        L.ref_state_hash.restype = C.c_uint64
        L.ref_verify_exact_cover.argtypes = [C.c_int, C.c_int64, _u32p, C.c_uint64,
                                             C.POINTER(C.c_int), _i64p, _u64p]
        L.ref_map_outcomes_t.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, _i64p, C.c_uint64]
        L.ref_decompose_trapezoids.argtypes = [C.c_int64, C.c_int64, _i64p, C.c_int, C.POINTER(C.c_int)]
        L.ref_map_trapezoid.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_int64, C.c_int64, _i64p]
        L.ref_make_edm_points.argtypes = [C.c_int64, C.c_uint64, _f64p]
        L.ref_kernel_edm.argtypes = [C.c_int64, C.c_uint64, _f64p, C.c_uint64, _u64p]
        L.ref_launch_edm.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, _f64p, C.c_uint64,
                                     _u64p, _u64p]
        L.ref_csv_optimize.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_char_p, C.c_uint64,
                                       C.POINTER(C.c_uint64)]
        L.ref_csv_sweep.argtypes = [C.c_int, C.c_int, C.c_char_p, C.c_int64, C.c_int64, C.c_int, C.c_char_p,
                                    C.c_uint64, C.POINTER(C.c_uint64), C.c_char_p, C.c_uint64]
        self.L = L

    def _ok(self, rc: int, what: str) -> None:
        if rc != 0:
            raise OracleError(f"{what}: status {rc}: {self.L.ref_last_error().decode()}")

    def make_grid(self, kind: int, m: int, n: int, rho: int = 1, T: int = 1):
        e = np.zeros(3, np.int64)
        b = np.zeros(1, np.uint64)
        ds = np.zeros(1, np.int64)
        self._ok(self.L.ref_make_grid(kind, m, n, rho, T, e, b, ds), "make_grid")
        return tuple(int(v) for v in e), int(b[0]), int(ds[0])

    def map_outcomes(self, kind: int, m: int, n: int, T: int = 1) -> np.ndarray:
        (ex, ey, ez), blocks, _ = self.make_grid(kind, m, n, 1, T)
        out = np.zeros((blocks, 6), np.int64)
        self._ok(self.L.ref_map_outcomes_t(kind, m, n, T, out, blocks), "map_outcomes")
        return out

    def csv_optimize(self, m: int, inv_r_max: int, beta_max: int, n_eval: int) -> str:
        cap = 1 << 20
        buf = C.create_string_buffer(cap)
        n = C.c_uint64(0)
        rc = self.L.ref_csv_optimize(m, inv_r_max, beta_max, n_eval, buf, cap, C.byref(n))
        if rc == 1:
            raise ValueError(self.L.ref_last_error().decode())
        self._ok(rc, "csv_optimize")
        return buf.raw[:n.value].decode()

    def csv_sweep(self, kind: int, m: int, nrange: str, rho: int = 1, T: int = 1, analyze: bool = False):
        """verify_sweep + csv_measure (or analyze_sweep + csv_analyze); -> (text, witnesses)"""
        cap = 1 << 24
        buf = C.create_string_buffer(cap)
        wbuf = C.create_string_buffer(1 << 16)
        n = C.c_uint64(0)
        self._ok(self.L.ref_csv_sweep(kind, m, nrange.encode(), rho, T, 1 if analyze else 0, buf, cap, C.byref(n),
                                      wbuf, 1 << 16), "csv_sweep")
        return buf.raw[:n.value].decode(), wbuf.value.decode()

    def make_edm_points(self, count: int, seed: int) -> np.ndarray:
        out = np.zeros((count, 2), np.float64)
        self._ok(self.L.ref_make_edm_points(count, seed, out), "make_edm_points")
        return out

    def kernel_edm(self, side: int, seed: int):
        cells = np.zeros(tri_cells(side), np.float64)
        h = np.zeros(1, np.uint64)
        self._ok(self.L.ref_kernel_edm(side, seed, cells, cells.size, h), "kernel_edm")
        return cells, int(h[0])

    def launch_edm(self, kind: int, n: int, rho: int, seed: int, T: int = 1):
        _, _, ds = self.make_grid(kind, 2, n, rho, T)
        side = ds * rho
        cells = np.zeros(tri_cells(side), np.float64)
        cnt = np.zeros(6, np.uint64)
        h = np.zeros(1, np.uint64)
        self._ok(self.L.ref_launch_edm(kind, n, rho, T, seed, cells, cells.size, cnt, h), "launch_edm")
        return cells, [int(v) for v in cnt], int(h[0])

    def decompose_trapezoids(self, n: int, T: int) -> list[dict]:
        out = np.zeros(9 * 64, np.int64)
        c = C.c_int(0)
        rc = self.L.ref_decompose_trapezoids(n, T, out, 64, C.byref(c))
        if rc == 1:
            raise ValueError(self.L.ref_last_error().decode())
        self._ok(rc, "decompose_trapezoids")
        keys = ("delta_x", "delta_y", "band", "h1", "h2", "grid_width", "valid_side", "ext_x", "ext_y")
        return [dict(zip(keys, (int(v) for v in out[9 * i:9 * i + 9]))) for i in range(c.value)]

    def map_trapezoid(self, n: int, T: int, band: int, x: int, y: int):
        o = np.zeros(6, np.int64)
        rc = self.L.ref_map_trapezoid(n, T, band, x, y, o)
        if rc == 1:
            raise ValueError(self.L.ref_last_error().decode())
        self._ok(rc, "map_trapezoid")
        return tuple(int(v) for v in o)

    def map_one(self, kind: int, m: int, n: int, x: int, y: int, z: int = 0):
        o = np.zeros(6, np.int64)
        rc = self.L.ref_map_one(kind, m, n, x, y, z, o)
        if rc == 1:
            raise ValueError(self.L.ref_last_error().decode())
        self._ok(rc, "map_one")
        return tuple(int(v) for v in o)

    def launch_map(self, kind: int, m: int, n: int, rho: int = 1, T: int = 1,
                   coverage: bool = True, salt: int = 0):
        _, _, ds = self.make_grid(kind, m, n, rho, T)
        side = ds * rho
        cov = np.zeros(cells_of(m, side), np.uint32) if coverage else None
        cnt = np.zeros(6, np.uint64)
        self._ok(self.L.ref_launch_map(kind, m, n, rho, T,
                                       cov.ctypes.data if cov is not None else None,
                                       cells_of(m, side), salt, cnt), "launch_map")
        return cov, [int(v) for v in cnt]

    def launch_accum(self, kind: int, m: int, n: int, rho: int, passes: int = 1,
                     cells: np.ndarray | None = None, T: int = 1):
        _, _, ds = self.make_grid(kind, m, n, rho, T)
        side = ds * rho
        if cells is None:
            cells = np.zeros(cells_of(m, side), np.uint32)
        cnt = np.zeros(6, np.uint64)
        h = np.zeros(1, np.uint64)
        secs = C.c_double(0.0)
        self._ok(self.L.ref_launch_accum(kind, m, n, rho, T, passes, cells, cells.size, cnt, h,
                                         C.byref(secs)), "launch_accum")
        return cells, [int(v) for v in cnt], int(h[0]), secs.value

    def accum_sample(self, kind: int, m: int, n: int, rho: int, rows: int, threads: int, warm: int = 1,
                     reps: int = 1):
        """ref_accum_sample: the reference's launch_accum sweep over the first
        `rows` block rows of the grid, `threads` concurrent replicas. Returns
        (seconds per rep [reps], useful cells per replica per rep)."""
        secs = np.zeros(reps, np.float64)
        useful = np.zeros(1, np.uint64)
        self._ok(self.L.ref_accum_sample(kind, m, n, rho, rows, threads, warm, reps, secs, useful),
                 "accum_sample")
        return secs.tolist(), int(useful[0])

    def make_life_state(self, m: int, side: int, seed: int) -> np.ndarray:
        out = np.empty(cells_of(m, side), np.uint8)
        self._ok(self.L.ref_make_life_state(m, side, seed, out, out.size), "make_life_state")
        return out

    def kernel_ca_run(self, m: int, side: int, steps: int, cells: np.ndarray):
        secs = C.c_double(0.0)
        self._ok(self.L.ref_kernel_ca_run(m, side, steps, cells, cells.size, C.byref(secs)),
                 "kernel_ca_run")
        return cells, secs.value

    def launch_ca(self, kind: int, m: int, n: int, rho: int, steps: int, cells: np.ndarray,
                  T: int = 1):
        cnt = np.zeros(6, np.uint64)
        h = np.zeros(1, np.uint64)
        secs = C.c_double(0.0)
        self._ok(self.L.ref_launch_ca(kind, m, n, rho, T, steps, cells, cells.size, cnt, h,
                                      C.byref(secs)), "launch_ca")
        return cells, [int(v) for v in cnt], int(h[0]), secs.value

    def state_hash(self, m: int, side: int, arr: np.ndarray) -> int:
        a = np.ascontiguousarray(arr)
        return int(self.L.ref_state_hash(m, side, a.ctypes.data, a.nbytes))

    def verify_exact_cover(self, m: int, side: int, cov: np.ndarray):
        exact = C.c_int(0)
        w = np.zeros(3, np.int64)
        mult = np.zeros(1, np.uint64)
        self._ok(self.L.ref_verify_exact_cover(m, side, cov, cov.size, C.byref(exact), w, mult),
                 "verify_exact_cover")
        return bool(exact.value), tuple(int(v) for v in w), int(mult[0])


def reference_available() -> bool:
    return os.path.exists(REF_SO)
