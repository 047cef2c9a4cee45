"""smx_ca_multi host-overhead probe: a small state (H3D(32) rho=8, side 248),
8 shards on one GPU, 100 steps: with the step-pair graph vs steps issued one
by one (SMX_MULTI_NOGRAPH=1)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2208_11617_b200 import api  # noqa: E402
g = api.make_grid(api.map_kind.h3d, 3, 32, 8)
side = g.cell_side()
a = torch.empty(api.tet_cells(side) + 256, dtype=torch.uint8, device="cuda")[:api.tet_cells(side)]
out = {}
for k in (2, 8):
    ms = []
    for i in range(4):
        api.life_init_device(3, side, 42, a)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); api.ca_multi(g, a, 100, [0] * k); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    out[f"shards_{k}_us_per_step"] = round(10 * statistics.median(ms[1:]), 2)
print(json.dumps({"graph": os.environ.get("SMX_MULTI_NOGRAPH") is None, **out}))
