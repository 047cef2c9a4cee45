"""GPU verification sweeps + CSV emitters: byte-identical to
the reference's verify_sweep/analyze_sweep + csv_measure/csv_analyze
(report.hpp:324-412), and the reference's trapezoid acceptance sweep
(acceptance.cpp:108-125: all n in [2, 4096], T in {1, 4, 16}) on the GPU."""
import pytest

from oracle.oracle import BB, H2D, H3D, LAMBDA, PADDED, RB, TRAP
from paper_2208_11617_b200 import api
from paper_2208_11617_b200 import report as rp

pytestmark = pytest.mark.gpu

SWEEPS = [(H2D, 2, "2..1024(pow2)", 1, 1), (H2D, 2, "2..256(pow2)", 3, 1), (TRAP, 2, "2..300", 1, 4),
          (TRAP, 2, "2..64", 2, 1), (PADDED, 2, "2..200", 1, 1), (RB, 2, "1..100", 1, 1), (LAMBDA, 2, "1..60", 2, 1),
          (BB, 2, "1..80", 1, 1), (BB, 3, "1..20", 2, 1), (H3D, 3, "4..64(pow2)", 2, 1)]


@pytest.mark.parametrize("kind,m,nr,rho,T", SWEEPS)
def test_csv_byte_identical_to_reference(cuda, ref, kind, m, nr, rho, T):
    ns = rp.expand_n_range(rp.parse_n_range(nr))
    want, witnesses = ref.csv_sweep(kind, m, nr, rho, T)
    rows = rp.verify_sweep(kind, m, ns, rho, T)
    assert rp.csv_measure(rows) == want
    assert all(r.exact for r in rows) and witnesses == ""
    want_an, _ = ref.csv_sweep(kind, m, nr, rho, T, analyze=True)
    assert rp.csv_analyze(rp.analyze_sweep(kind, m, ns, rho, T)) == want_an


def test_trapezoid_acceptance_sweep(cuda):
    # acceptance.cpp:108-125 (criterion 4): exact for every n in [2, 4096], T in
    # {1, 4, 16}, with at most ceil(log2 n) bands
    for T in (1, 4, 16):
        rows = rp.verify_sweep(api.map_kind.h2d_trapezoid, 2, list(range(2, 4097)), 1, T)
        assert all(r.exact for r in rows), [(r.n, rp.witness_text(r)) for r in rows if not r.exact][:3]
        for r in rows:
            assert len(api.decompose_trapezoids(r.n, T)) <= max(1, (r.n - 1).bit_length())


def test_witness_on_planted_defect(cuda):
    import torch
    g = api.grid_h2d(16)
    side = g.cell_side()
    cov = torch.zeros(api.tri_cells(side), dtype=torch.int32, device="cuda")
    api.launch_map_device(g, cov)
    cov[api.tri_linear_index(3, 7)] += 1
    import ctypes as C
    first, mult = C.c_uint64(0), C.c_uint32(0)
    api.check(api.lib().smx_verify_cover(api._ptr(cov), cov.numel(), 1, C.byref(first), C.byref(mult),
                                         api._stream()))
    assert first.value == api.tri_linear_index(3, 7) and mult.value == 2
