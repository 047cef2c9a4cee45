timeout 900 python -m pytest tests/test_gpu_ca.py -x -q 2>&1 | tail -2
for c in "h3d 64 4" "h3d 128 8" "h3d 256 8" "bb 255 8"; do timeout 120 python tools/prof_case.py ca $c bits 6 | sed 's/, all=.*//'; done
python - <<'PY' > gpurun_out/prof2_cases.txt 2>&1
import torch, sys
sys.path.insert(0, '.')
from paper_2208_11617_b200 import api
g = api.make_grid(api.map_kind.h2d, 2, 1024, 16); side = g.cell_side(); n = api.tri_cells(side)
pts = torch.from_numpy(api.make_edm_points(side, 7)).cuda(); e = torch.empty(n, dtype=torch.float64, device='cuda')
a = torch.empty(n, dtype=torch.uint8, device='cuda'); b = torch.empty_like(a); api.life_init_device(2, side, 42, a)
gt = api.make_grid(api.map_kind.h2d_trapezoid, 2, 4097, 16, 4); ct = torch.zeros(api.tri_cells(gt.cell_side()), dtype=torch.int32, device='cuda')
for i in range(3):
    api.edm_device(g, pts, e, api.EXEC_RUNS); api.ca_step_device(g, a, b, api.EXEC_RUNS); api.accum_device(gt, ct, 1, api.EXEC_RUNS)
torch.cuda.synchronize(); print("ok")
PY
cat > /tmp/p2.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
from paper_2208_11617_b200 import api
g = api.make_grid(api.map_kind.h2d, 2, 1024, 16); side = g.cell_side(); n = api.tri_cells(side)
pts = torch.from_numpy(api.make_edm_points(side, 7)).cuda(); e = torch.empty(n, dtype=torch.float64, device='cuda')
a = torch.empty(n, dtype=torch.uint8, device='cuda'); b = torch.empty_like(a); api.life_init_device(2, side, 42, a)
gt = api.make_grid(api.map_kind.h2d_trapezoid, 2, 4097, 16, 4); ct = torch.zeros(api.tri_cells(gt.cell_side()), dtype=torch.int32, device='cuda')
for i in range(3):
    api.edm_device(g, pts, e, api.EXEC_RUNS); api.ca_step_device(g, a, b, api.EXEC_RUNS); api.accum_device(gt, ct, 1, api.EXEC_RUNS)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_edm_runs|k_ca2d_runs|k_accum_runs" -s 3 -c 3 -o gpurun_out/rows_f python /tmp/p2.py > /dev/null 2>&1; echo "ncu rc=$?"
