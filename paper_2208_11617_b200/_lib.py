"""ctypes binding of the C ABI (include/smx_b200.h) in libsmx_b200.so.

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the shared object is missing or fails to load, every
entry point raises ``RuntimeError`` naming the build command.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsmx_b200.so")

SMX_OK, SMX_EINVAL, SMX_ERANGE, SMX_ECUDA, SMX_ENOMEM = 0, 1, 2, 3, 4
EXEC_AUTO, EXEC_BLOCK, EXEC_RUNS, EXEC_BITS = -1, 0, 1, 2


class smx_grid(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("dims", C.c_int32),
        ("n", C.c_int64),
        ("rho", C.c_int64),
        ("threshold", C.c_int64),
        ("extents", C.c_int64 * 3),
    ]


class smx_counters(C.Structure):
    _fields_ = [
        ("blocks_launched", C.c_uint64),
        ("blocks_void", C.c_uint64),
        ("threads_launched", C.c_uint64),
        ("threads_useful", C.c_uint64),
    ]


class smx_outcome(C.Structure):
    _fields_ = [
        ("is_void", C.c_int32),
        ("x", C.c_int32),
        ("y", C.c_int32),
        ("z", C.c_int32),
        ("level_b", C.c_int32),
        ("index_q", C.c_int32),
        ("pad0", C.c_int32),
        ("pad1", C.c_int32),
    ]


class smx_trapezoid(C.Structure):
    _fields_ = [(f, C.c_int64) for f in ("delta_x", "delta_y", "band", "h1", "h2", "grid_width", "valid_side",
                                         "ext_x", "ext_y")]


_G = C.POINTER(smx_grid)
_VP = C.c_void_p
_SIGS = {
    "smx_last_error": ([], C.c_char_p),
    "smx_make_grid": ([C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_int64, _G], C.c_int),
    "smx_cell_side": ([_G], C.c_int64),
    "smx_cell_count": ([C.c_int32, C.c_int64], C.c_uint64),
    "smx_map_one": ([C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                     C.POINTER(smx_outcome)], C.c_int),
    "smx_map_outcomes": ([_G, _VP, C.c_uint64, C.c_int, _VP], C.c_int),
    "smx_launch_map": ([_G, _VP, C.c_uint64, C.c_int, C.POINTER(smx_counters), _VP], C.c_int),
    "smx_map_kernel": ([_G, _VP], C.c_int),
    "smx_accum": ([_G, _VP, C.c_uint64, C.c_int64, C.c_int32, C.c_int, _VP,
                   C.POINTER(smx_counters), _VP], C.c_int),
    "smx_accum_range": ([_G, _VP, C.c_uint64, C.c_int64, C.c_int32, C.c_int64, C.c_int64,
                         C.POINTER(smx_counters), _VP], C.c_int),
    "smx_life_init": ([C.c_int32, C.c_int64, C.c_uint64, _VP, C.c_uint64, C.c_int, _VP], C.c_int),
    "smx_ca_step": ([_G, _VP, _VP, C.c_uint64, C.c_int32, _VP], C.c_int),
    "smx_ca": ([_G, _VP, C.c_uint64, C.c_int64, C.c_int32, C.c_int, _VP, _VP,
                C.POINTER(smx_counters), _VP], C.c_int),
    "smx_state_hash": ([C.c_int32, C.c_int64, _VP, C.c_uint64], C.c_uint64),
    "smx_ca_step_range": ([_G, _VP, _VP, C.c_uint64, C.c_int64, C.c_int64, C.c_int32, _VP], C.c_int),
    "smx_tile_bytes": ([_G, C.c_uint64], C.c_uint64),
    "smx_tiles_pack": ([_G, _VP, _VP, C.c_uint64, _VP, _VP], C.c_int),
    "smx_tiles_unpack": ([_G, _VP, _VP, C.c_uint64, _VP, _VP], C.c_int),
    "smx_device_sync": ([], C.c_int),
    "smx_release": ([], C.c_int),
    "smx_ca_engine": ([_G], C.c_int),
    "smx_ca_multi": ([_G, _VP, C.c_uint64, C.c_int64, _VP, C.c_int32, C.c_int, _VP, _VP], C.c_int),
    "smx_bits_plan_capacity": ([_G], C.c_uint64),
    "smx_bits_plan": ([_G, C.c_int64, C.c_int64, _VP, _VP, _VP], C.c_int),
    "smx_bits_run_list": ([_G, _VP, _VP, _VP, _VP, _VP], C.c_int),
    "smx_kernel_accum": ([_VP, C.c_uint64, C.c_int, _VP], C.c_int),
    "smx_kernel_edm": ([_VP, C.c_int64, _VP, C.c_uint64, C.c_int, _VP], C.c_int),
    "smx_kernel_ca_run": ([C.c_int32, C.c_int64, _VP, C.c_uint64, C.c_int64, C.c_int, _VP], C.c_int),
    "smx_scratch_bytes": ([], C.c_uint64),
    "smx_bits_bytes": ([_G], C.c_uint64),
    "smx_bits_pack": ([_G, _VP, C.c_uint64, _VP, _VP], C.c_int),
    "smx_bits_step": ([_G, _VP, _VP, C.c_int64, C.c_int64, _VP], C.c_int),
    "smx_bits_unpack": ([_G, _VP, _VP, C.c_uint64, _VP], C.c_int),
    "smx_bits_run": ([_G, _VP, _VP, C.c_int64, _VP], C.c_int),
    "smx_grid_blocks": ([_G], C.c_uint64),
    "smx_make_edm_points": ([C.c_int64, C.c_uint64, _VP], C.c_int),
    "smx_bits_tile_bytes": ([_G, C.c_uint64], C.c_uint64),
    "smx_bits_tiles_pack": ([_G, _VP, _VP, C.c_uint64, _VP, _VP], C.c_int),
    "smx_bits_tiles_unpack": ([_G, _VP, _VP, C.c_uint64, _VP, _VP], C.c_int),
    "smx_measure_grid": ([_G, C.c_int, _VP, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), _VP], C.c_int),
    "smx_verify_cover": ([_VP, C.c_uint64, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), _VP], C.c_int),
    "smx_edm": ([_G, _VP, C.c_int64, _VP, C.c_uint64, C.c_int32, C.c_int, _VP, _VP, _VP], C.c_int),
    "smx_decompose_trapezoids": ([C.c_int64, C.c_int64, C.POINTER(smx_trapezoid), C.c_int32,
                                  C.POINTER(C.c_int32)], C.c_int),
    "smx_map_trapezoid": ([C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.POINTER(smx_outcome)],
                          C.c_int),
}

_lib = None


def lib() -> C.CDLL:
    """Load libsmx_b200.so (once). Raises if it was never built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the sm_100a library with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class Overflow(OverflowError):
    """std::overflow_error in the reference."""


class CudaError(RuntimeError):
    pass


def check(rc: int) -> None:
    if rc == SMX_OK:
        return
    msg = lib().smx_last_error().decode()
    if rc == SMX_EINVAL:
        raise InvalidArgument(msg)
    if rc == SMX_ERANGE:
        raise Overflow(msg)
    raise CudaError(f"smx error {rc}: {msg}")
