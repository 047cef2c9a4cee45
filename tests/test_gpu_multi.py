"""smx_ca_multi — launch_ca over several GPUs of ONE process (the C ABI's
multi-GPU path): whole-H-level shards, per-shard engine plan
split into boundary / interior chunks, bit-tile halo by peer copies while the
interior runs. This box has one GPU, so the shards share cuda:0 (the same
schedule; the peer copies are local), which exercises the partition, the
halo plan, the chunk split and the stream/event ordering exactly."""
import numpy as np
import pytest

from conftest import golden
from paper_2208_11617_b200 import api

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,n,rho,shards", [("h3d", 32, 8, 2), ("h3d", 32, 8, 3), ("h3d", 64, 4, 4),
                                                ("bb", 31, 8, 2), ("bb", 63, 4, 5), ("h3d", 16, 4, 6)])
def test_multi_vs_oracle(cuda, orc, kind, n, rho, shards):
    g = api.make_grid(api.map_kind[kind], 3, n, rho)
    side = g.cell_side()
    steps = 7
    want = orc.make_life_state(3, side, 42)
    orc.ca3d_run(side, steps, want)
    # host state through the Python launch_ca (opts.devices), report as single-GPU
    st = api.make_life_state(3, side, 42)
    rep = api.launch_ca(g, api.simplex_spec(3, side - 1), st,
                        api.launch_opts(steps=steps, boundary=api.ca_boundary.dead3d, devices=(0,) * shards))
    assert (st.cells == want).all(), (kind, n, rho, shards)
    assert rep.threads_useful == api.tet_cells(side)
    assert api.verify_exact_cover(rep, api.simplex_spec(3, side - 1)).exact
    # device state, twice (the cached plan and replicas are reused)
    import torch
    for _ in range(2):
        a = torch.empty(api.tet_cells(side), dtype=torch.uint8, device="cuda")
        api.life_init_device(3, side, 42, a)
        api.ca_multi(g, a, steps, [0] * shards)
        assert (a.cpu().numpy() == want).all()


@pytest.mark.slow
def test_multi_c4_golden(cuda):
    """C4 (H3D(128), rho = 8), 100 steps on 4 and 8 shards = the oracle golden."""
    import torch
    want = golden("ca_full.json")["cases"]["c4_rho8_100"]
    g = api.make_grid(api.map_kind.h3d, 3, 128, 8)
    side = g.cell_side()
    for shards in (4, 8):
        a = torch.empty(api.tet_cells(side), dtype=torch.uint8, device="cuda")
        api.life_init_device(3, side, 42, a)
        api.ca_multi(g, a, 100, [0] * shards)
        assert api.state_hash(3, side, a.cpu().numpy()) == int(want["final_hash"]), shards
    api.release_scratch()


def test_multi_errors(cuda):
    g = api.make_grid(api.map_kind.h3d, 3, 16, 8)
    st = api.make_life_state(3, g.cell_side(), 1)
    with pytest.raises(api.InvalidArgument):
        api.ca_multi(g, st.cells, 1, [0, 99])
    with pytest.raises(api.InvalidArgument):
        api.ca_multi(g, st.cells, -1, [0])
    g2 = api.make_grid(api.map_kind.h2d, 2, 16, 8)
    st2 = api.make_life_state(2, g2.cell_side(), 1)
    with pytest.raises(api.InvalidArgument):
        api.ca_multi(g2, st2.cells, 1, [0, 0])
    assert np.asarray(st.cells).size == api.tet_cells(g.cell_side())
