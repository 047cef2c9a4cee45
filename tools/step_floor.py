"""Per-step cost of the persistent CA engine vs grid size (slope between a 10-
and a 110-step smx_bits_run launch), down to a nearly empty grid: the fixed
per-step latency (grid barrier + one item) the small configs run into."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2208_11617_b200 import api  # noqa: E402


def t(fn, it=5):
    ms = []
    for _ in range(it):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ms.append(s.elapsed_time(e))
    return statistics.median(ms[1:])


for kind, n, rho in [("h3d", 4, 4), ("h3d", 8, 4), ("h3d", 16, 4), ("h3d", 32, 4), ("h3d", 64, 4), ("bb", 63, 4),
                     ("h3d", 16, 8), ("h3d", 32, 8), ("h3d", 64, 8), ("h3d", 128, 8)]:
    g = api.make_grid(api.map_kind[kind], 3, n, rho)
    side = g.cell_side()
    cells = api.tet_cells(side)
    a = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
    api.life_init_device(3, side, 42, a)
    sa, sb = api.bits_buffer(g), api.bits_buffer(g)
    api.bits_pack_device(g, a, sa)
    t10 = t(lambda: api.bits_run_device(g, sa, sb, 10))
    t110 = t(lambda: api.bits_run_device(g, sa, sb, 110))
    per = (t110 - t10) / 100
    print(f"{kind}({n}) rho={rho} side={side} cells={cells}: per step {per * 1000:.2f} us "
          f"({cells / per / 1e6:.1f} Gcell-steps/s), fixed {t10 - 10 * per:.4f} ms")
