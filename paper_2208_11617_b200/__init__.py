"""B200-native (sm_100a) H block-space maps for 2- and 3-simplex domains
(arXiv 2208.11617), behind the reference `simplexmap` hot-path API.

    from paper_2208_11617_b200 import api
    g = api.grid_h2d(1024); g.rho = 16
    st = api.simplex_grid_state(2, g.cell_side())
    rep = api.launch_accum(g, api.simplex_spec(2, g.cell_side() - 1), st)

The compute path is libsmx_b200.so (C ABI in include/smx_b200.h); see
DESIGN.md for the kernels and INTEGRATION.md for the reference-side bindings.
"""
from . import _lib  # noqa: F401

__all__ = ["api", "dist"]
