"""One engine launch for ncu (run on the GPU box):
    SMX_CA_ENGINE=cols ncu ... python tools/prof_engine.py h3d 256 8 2
Warms up once, then runs smx_bits_run for `steps` steps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2208_11617_b200 import api  # noqa: E402

kind, n, rho, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
g = api.make_grid(api.map_kind[kind], 3, n, rho)
side = g.cell_side()
cells = api.tet_cells(side)
u8 = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
api.life_init_device(3, side, 42, u8)
A, B = api.bits_buffer(g), api.bits_buffer(g)
api.bits_pack_device(g, u8, A)
api.bits_run_device(g, A, B, steps)
torch.cuda.synchronize()
api.bits_run_device(g, A, B, steps)
torch.cuda.synchronize()
print("ok")
