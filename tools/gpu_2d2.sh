timeout 1500 python -m pytest tests/test_gpu_maps2d.py -x -q 2>&1 | tail -6
python - <<'PY'
import statistics, torch, sys
sys.path.insert(0, '.')
from paper_2208_11617_b200 import api
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
def tm(fn, iters=6):
    ms=[]
    for i in range(iters):
        flush.fill_(i)
        s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ms.append(s.elapsed_time(e))
    return statistics.median(ms[1:])
for kind,n in ((api.map_kind.h2d,1024),(api.map_kind.bb,1023),(api.map_kind.h2d_trapezoid,1000)):
    g = api.make_grid(kind,2,n,16,1); side=g.cell_side(); cells=api.tri_cells(side)
    pts = torch.from_numpy(api.make_edm_points(side, 1)).cuda()
    out = torch.empty(cells, dtype=torch.float64, device='cuda')
    for ex,name in ((api.EXEC_RUNS,'runs'),(api.EXEC_BLOCK,'block')):
        m = tm(lambda: api.edm_device(g, pts, out, ex))
        print(f"EDM {g} {name}: {m:.4f} ms {cells/m/1e6:.1f} Gcells/s {8*cells/m/1e6:.0f} GB/s")
    a = torch.zeros(cells, dtype=torch.uint8, device='cuda'); api.life_init_device(2, side, 42, a); b = torch.empty_like(a)
    for ex,name in ((api.EXEC_RUNS,'runs'),(api.EXEC_BLOCK,'block')):
        m = tm(lambda: api.ca_step_device(g, a, b, ex))
        print(f"CA2D {g} {name}: {m:.4f} ms {cells/m/1e6:.1f} Gcells/s {2*cells/m/1e6:.0f} GB/s")
PY
