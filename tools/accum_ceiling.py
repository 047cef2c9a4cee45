import sys, statistics, json
sys.path.insert(0, '/root/repo')
import torch, ctypes as C
from paper_2208_11617_b200 import api, _lib
L = _lib.lib()
g = api.make_grid(api.map_kind.h2d, 2, 4096, 16)
cells = api.tri_cells(g.cell_side())
a = torch.zeros(cells, dtype=torch.int32, device='cuda')
def t(fn, n=10):
    for _ in range(3): fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for e0, e1 in ev:
        e0.record(); fn(); e1.record()
    torch.cuda.synchronize()
    return statistics.median(e0.elapsed_time(e1) for e0, e1 in ev)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
res = {}
res['accum_runs_ms'] = t(lambda: api.accum_device(g, a, 1, api.EXEC_RUNS))
gb = api.make_grid(api.map_kind.bb, 2, 4095, 16)
res['accum_runs_bb_ms'] = t(lambda: api.accum_device(gb, a, 1, api.EXEC_RUNS))
res['kernel_accum_ms'] = t(lambda: _lib.check(L.smx_kernel_accum(C.c_void_p(a.data_ptr()), cells, 1, s)))
b = torch.empty_like(a)
res['torch_copy_ms'] = t(lambda: b.copy_(a))
res['torch_add_inplace_ms'] = t(lambda: a.add_(1))
for k in list(res): res[k.replace('_ms','_gbs')] = round(8 * cells / (res[k] * 1e-3) / 1e9, 1)
print(json.dumps(res))
