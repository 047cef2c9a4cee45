"""Reentrancy of the C ABI (include/smx_b200.h "Threads"): the reference's
launch_* functions are pure and may run concurrently on distinct states
(simulator.hpp:313-326,431-463). Two host threads, each on its own CUDA stream,
run launch_ca (host buffers, the bit-shadow engine: pack, side-stream plan,
persistent run, unpack) on different grids at the same time, repeatedly; every
result must equal the restated oracle's sequential run."""
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
            with torch.cuda.stream(torch.cuda.Stream()):
                g = api.make_grid(kind, 3, n, rho)
                side = g.cell_side()
                barrier.wait()
                for _ in range(12):
                    st = api.make_life_state(3, side, seed)
                    api.launch_ca(g, api.simplex_spec(3, side - 1), st,
                                  api.launch_opts(steps=steps, boundary=api.ca_boundary.dead3d,
                                                  exec=api.EXEC_BITS, record_coverage=False))
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
