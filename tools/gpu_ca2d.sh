# 2-D periodic Life: parity (GPU tests) + one-step timing of the x-run kernel
# at F3's shape and a larger one, + ncu capture of the kernel.
timeout 900 python -m pytest tests/test_gpu_maps2d.py tests/test_dropin_cpp.py -x -q 2>&1 | tail -4
python - <<'PY'
import statistics, torch, sys
sys.path.insert(0, '.')
from paper_2208_11617_b200 import api
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
def t(g, ex, iters=10):
    side = g.cell_side(); cells = api.tri_cells(side)
    a = torch.empty(cells, dtype=torch.uint8, device='cuda'); b = torch.empty_like(a)
    api.life_init_device(2, side, 42, a)
    ms = []
    for i in range(iters):
        flush.fill_(i)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); api.ca_step_device(g, a, b, ex); e.record(); torch.cuda.synchronize(); ms.append(s.elapsed_time(e))
    m = statistics.median(ms[2:])
    print(f"{g} ex={ex}: {m*1e3:.1f} us {cells/m/1e6:.1f} Gcells/s frac(2B/cell, 6650)={2*cells/m/1e6/6650:.3f}")
for g in (api.make_grid(api.map_kind.h2d, 2, 1024, 16), api.make_grid(api.map_kind.bb, 2, 1023, 16),
          api.make_grid(api.map_kind.h2d, 2, 4096, 16), api.make_grid(api.map_kind.h2d, 2, 4096, 4),
          api.make_grid(api.map_kind.h2d, 2, 65536, 1), api.make_grid(api.map_kind.rb, 2, 4095, 16)):
    t(g, api.EXEC_RUNS)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ca2d_" -s 2 -c 1 -o gpurun_out/ca2d python tools/prof_case.py ca2d h2d 4096 16 runs 3 > /dev/null 2>&1; echo "ncu rc=$?"
