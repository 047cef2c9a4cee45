# EDM x-run timing (H2D(1024) rho=16, BB(1023), H2D(4096) rho=16) + parity
timeout 600 python -m pytest tests/test_gpu_maps2d.py -x -q -k edm 2>&1 | tail -1
python - <<'PY'
import sys, statistics, torch
sys.path.insert(0, '.')
from paper_2208_11617_b200 import api
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
for kind, n, rho in (("h2d", 1024, 16), ("bb", 1023, 16), ("h2d", 2048, 16)):
    g = api.make_grid(api.map_kind[kind], 2, n, rho); side = g.cell_side(); cells = api.tri_cells(side)
    pts = torch.from_numpy(api.make_edm_points(side, 7)).cuda(); e = torch.empty(cells, dtype=torch.float64, device='cuda')
    ms = []
    for i in range(8):
        flush.fill_(i); s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); api.edm_device(g, pts, e, api.EXEC_RUNS); t.record(); torch.cuda.synchronize(); ms.append(s.elapsed_time(t))
    m = statistics.median(ms[1:])
    print(f"edm {kind}({n}) rho={rho}: {m:.4f} ms, {cells/m/1e6:.1f} Gcells/s, {8*cells/m/1e6/6552.3:.3f} of peak")
    del e, pts; torch.cuda.empty_cache()
PY
