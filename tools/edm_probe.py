"""EDM x-run timing at C1 scale (H2D(1024) rho=16, side 16368): GB/s of f64 writes."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_11617_b200 import api  # noqa: E402

res = {}
for name, g in (("h", api.make_grid(api.map_kind.h2d, 2, 1024, 16)), ("bb", api.make_grid(api.map_kind.bb, 2, 1023, 16))):
    side = g.cell_side()
    cells = api.tri_cells(side)
    pts = torch.from_numpy(api.make_edm_points(side, 7)).cuda()
    e = torch.empty(cells, dtype=torch.float64, device="cuda")
    for _ in range(3):
        api.edm_device(g, pts, e, api.EXEC_RUNS)
    ms = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        api.edm_device(g, pts, e, api.EXEC_RUNS)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    m = statistics.median(ms)
    res[name] = {"ms": round(m, 4), "gcells_s": round(cells / m / 1e6, 1), "gb_s": round(8 * cells / m / 1e6, 1)}
print(json.dumps(res))
