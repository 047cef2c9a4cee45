timeout 1500 python -m pytest tests/test_gpu_maps2d.py tests/test_gpu_maps.py tests/test_gpu_accum.py tests/test_dropin_cpp.py -x -q 2>&1 | tail -6
for a in "h2d 4096 16" "bb 4095 16"; do timeout 120 python tools/prof_case.py accum $a runs 6 | sed 's/, all=.*//'; done
python - <<'PY'
import statistics, torch, sys
sys.path.insert(0, '.')
from paper_2208_11617_b200 import api
def t(g, iters=6):
    c = torch.zeros(api.tri_cells(g.cell_side()), dtype=torch.int32, device='cuda')
    ms=[]
    for i in range(iters):
        s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        s.record(); api.accum_device(g, c, 1, api.EXEC_RUNS); e.record(); torch.cuda.synchronize(); ms.append(s.elapsed_time(e))
    m=statistics.median(ms[1:]); cells=api.tri_cells(g.cell_side())
    print(f"{g}: {m:.4f} ms {cells/m/1e6:.1f} Gcells/s {8*cells/m/1e6:.0f} GB/s")
for g in (api.make_grid(api.map_kind.h2d_trapezoid,2,4097,16,4), api.make_grid(api.map_kind.h2d_trapezoid,2,3000,16,1),
          api.make_grid(api.map_kind.h2d_padded,2,3000,16), api.make_grid(api.map_kind.rb,2,3000,16), api.make_grid(api.map_kind.lambda2d,2,3000,16),
          api.make_grid(api.map_kind.bb,2,3000,16), api.make_grid(api.map_kind.h2d,2,4096,16)):
    t(g)
PY
