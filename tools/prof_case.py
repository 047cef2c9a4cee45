"""Run one hot-path case in isolation (for ncu / quick timing on the GPU box).

    python tools/prof_case.py ca  h3d 256 8 [runs|block] [iters]
    python tools/prof_case.py accum h2d 4096 16 [runs|block] [iters]
    python tools/prof_case.py map h3d 256 1
    python tools/prof_case.py ca2d h2d 4096 16 [runs|block] [iters]
    python tools/prof_case.py multi h3d 32 8 bits [iters]        (smx_ca_multi, 3 shards on one GPU)
    SMX_CA_ENGINE=cols python tools/prof_case.py engine h3d 32 8 bits 2   (the column engine)
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2208_11617_b200 import api  # noqa: E402


def main():
    what, kind, n, rho = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    ex = {"runs": api.EXEC_RUNS, "block": api.EXEC_BLOCK, "bits": api.EXEC_BITS}[sys.argv[5] if len(sys.argv) > 5 else "runs"]
    iters = int(sys.argv[6]) if len(sys.argv) > 6 else 5
    m = 2 if what in ("accum", "ca2d", "kaccum") or (what == "map" and kind == "h2d") else 3
    if what == "map" and kind == "bb" and len(sys.argv) > 7:
        m = int(sys.argv[7])
    g = api.make_grid(api.map_kind[kind], m, n, rho)
    side = g.cell_side()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    if what == "ca":
        cells = api.tet_cells(side)
        a = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
        b = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
        api.life_init_device(3, side, 42, a)
        bufs = [a, b]
        fn = lambda i: api.ca_step_device(g, bufs[i % 2], bufs[(i + 1) % 2], ex)  # noqa: E731
        cells_done = cells
    elif what == "engine":  # multi-step bit-shadow engine, K fused steps per call
        cells = api.tet_cells(side)
        a = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
        scratch = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
        api.life_init_device(3, side, 42, a)
        K = 10
        fn = lambda i: api.ca_device(g, a, K, ex, scratch)  # noqa: E731
        cells_done = cells * K
    elif what == "ca2d":
        cells = api.tri_cells(side)
        a = torch.empty(cells, dtype=torch.uint8, device="cuda")
        b = torch.empty_like(a)
        api.life_init_device(2, side, 42, a)
        bufs = [a, b]
        fn = lambda i: api.ca_step_device(g, bufs[i % 2], bufs[(i + 1) % 2], ex)  # noqa: E731
        cells_done = cells
    elif what == "multi":  # smx_ca_multi, three shards on this device, 3 steps per call
        cells = api.tet_cells(side)
        a = torch.empty(cells + 256, dtype=torch.uint8, device="cuda")[:cells]
        api.life_init_device(3, side, 42, a)
        fn = lambda i: api.ca_multi(g, a, 3, [0, 0, 0])  # noqa: E731
        cells_done = cells * 3
    elif what == "kaccum":  # kernel_accum (no map) on a host state
        st = api.simplex_grid_state(2, side)
        fn = lambda i: api.kernel_accum(st)  # noqa: E731
        cells_done = api.tri_cells(side)
    elif what == "accum":
        cells = api.tri_cells(side)
        a = torch.zeros(cells, dtype=torch.int32, device="cuda")
        fn = lambda i: api.accum_device(g, a, 1, ex)  # noqa: E731
        cells_done = cells
    else:
        fn = lambda i: api.map_kernel_device(g)  # noqa: E731
        cells_done = g.blocks()
    ms = []
    for i in range(iters):
        flush.fill_(i & 0xff)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn(i)
        e.record()
        torch.cuda.synchronize()
        ms.append(s.elapsed_time(e))
    t = statistics.median(ms[1:] if len(ms) > 1 else ms)
    print(f"{what} {kind}({n}) rho={rho} side={side}: median {t:.4f} ms, {cells_done / t / 1e6:.1f} G/s, all={['%.4f' % v for v in ms]}")


if __name__ == "__main__":
    main()
