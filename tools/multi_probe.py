"""smx_ca_multi on ONE GPU (shards share the device): per-step cost vs the
single-GPU engine at C4 (H3D(128) rho=8, 100 steps) — the host-side schedule's
overhead (launches, peer copies, events) on top of the shards' work."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2208_11617_b200 import api  # noqa: E402

g = api.make_grid(api.map_kind.h3d, 3, 128, 8)
side = g.cell_side()
cells = api.tet_cells(side)
a = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
b = torch.empty_like(a)
res = {}
for name, fn in [("engine", lambda: api.ca_device(g, a, 100, api.EXEC_AUTO, b))] + [
        (f"multi_{k}", (lambda k=k: api.ca_multi(g, a, 100, [0] * k))) for k in (1, 2, 4, 8)]:
    api.life_init_device(3, side, 42, a)
    fn()
    ms = []
    for _ in range(3):
        api.life_init_device(3, side, 42, a)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    res[name] = {"ms_per_call": round(statistics.median(ms), 3), "us_per_step": round(10 * statistics.median(ms), 2)}
print(json.dumps(res))
