"""Reentrancy of the C ABI (include/smx_b200.h "Threads"): the reference's
launch_* functions are pure and may run concurrently on distinct states
(simulator.hpp:313-326,431-463). Two host threads, each on its own CUDA stream
(passed through launch_ca's `stream`), run launch_ca (host buffers, the
bit-shadow engine: staging copies, pack, side-stream plan, persistent run,
unpack) on different grids at the same time, repeatedly; every result must
equal the restated oracle's sequential run. The library orders the two
persistent whole-device grids per device; everything else overlaps. Each
thread's scratch is freed when it exits."""
import threading

import numpy as np
import pytest

from oracle.oracle import BB, H3D
from paper_2208_11617_b200 import api

pytestmark = pytest.mark.gpu


def test_concurrent_launch_ca_from_two_threads(cuda, orc):
    import torch

    cases = [(H3D, 16, 4, 11), (BB, 15, 8, 12)]  # kind, n, rho, seed
    steps = 6
    want = {}
    for kind, n, rho, seed in cases:
        side = api.make_grid(kind, 3, n, rho).cell_side()
        st = orc.make_life_state(3, side, seed)
        orc.ca3d_run(side, steps, st)
        want[seed] = st
    errors = []
    barrier = threading.Barrier(len(cases))

    def worker(kind, n, rho, seed):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                g = api.make_grid(kind, 3, n, rho)
                side = g.cell_side()
                barrier.wait()
                for _ in range(12):
                    st = api.make_life_state(3, side, seed)
                    api.launch_ca(g, api.simplex_spec(3, side - 1), st,
                                  api.launch_opts(steps=steps, boundary=api.ca_boundary.dead3d,
                                                  exec=api.EXEC_BITS, record_coverage=False),
                                  stream=stream)
                    if not np.array_equal(st.cells, want[seed]):
                        errors.append((kind, n, rho, seed))
                        return
        except Exception as e:  # noqa: BLE001 - surfaced through the assert below
            errors.append(repr(e))

    ts = [threading.Thread(target=worker, args=c) for c in cases]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_release_and_thread_exit_free_scratch(cuda):
    """smx_release frees the calling thread's pools; a worker thread's pools
    are freed when it exits (thread pools must not leak)."""
    import torch

    g = api.grid_h3d(64)  # side 504: ~80 MB of pools per thread
    g.rho = 8
    side = g.cell_side()
    st = api.make_life_state(3, side, 5)
    opts = api.launch_opts(steps=1, boundary=api.ca_boundary.dead3d, exec=api.EXEC_BITS, record_coverage=False)
    api.launch_ca(g, api.simplex_spec(3, side - 1), st, opts)
    assert api.scratch_bytes() > 0
    api.release_scratch()
    assert api.scratch_bytes() == 0
    free0 = torch.cuda.mem_get_info()[0]

    def worker():
        s2 = api.make_life_state(3, side, 5)
        api.launch_ca(g, api.simplex_spec(3, side - 1), s2, opts)

    for _ in range(6):
        t = threading.Thread(target=worker)
        t.start()
        t.join()
    torch.cuda.synchronize()
    # six exited workers hold nothing: free memory is back within 64 MiB.
    # Thread.join() can return before the native thread has run its TLS
    # destructors (Python releases the join lock first), so poll briefly.
    import time
    for _ in range(50):
        if torch.cuda.mem_get_info()[0] > free0 - (64 << 20):
            break
        time.sleep(0.1)
    assert torch.cuda.mem_get_info()[0] > free0 - (64 << 20)
