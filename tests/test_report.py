"""report layer host pieces against the reference: n-range
parsing (report.hpp:73-110), round-half-up decimals (rational.hpp:129-144)
checked on every row of reference-generated CSV, overhead limits (:345-352)."""
from fractions import Fraction

import pytest

from oracle.oracle import BB, H2D, H3D, PADDED, TRAP
from paper_2208_11617_b200 import api
from paper_2208_11617_b200 import report as rp


def test_n_range():
    assert rp.expand_n_range(rp.parse_n_range("7")) == [7]
    assert rp.expand_n_range(rp.parse_n_range("3..6")) == [3, 4, 5, 6]
    assert rp.expand_n_range(rp.parse_n_range("2..64(pow2)")) == [2, 4, 8, 16, 32, 64]
    assert rp.expand_n_range(rp.parse_n_range("3..100(pow2)")) == [4, 8, 16, 32, 64]
    assert rp.expand_n_range(rp.parse_n_range("1..1(pow2)")) == [1]
    for bad in ("", "x", "0..4", "5..4", "2..", "..3", "2..3(pow)"):
        with pytest.raises(api.InvalidArgument):
            rp.parse_n_range(bad)


def test_decimals_match_reference_csv(ref):
    for kind, m, nr, rho, T, an in [(H2D, 2, "2..1024(pow2)", 3, 1, False), (TRAP, 2, "2..120", 1, 4, True),
                                    (PADDED, 2, "2..90", 2, 1, False), (BB, 3, "1..25", 1, 1, True),
                                    (H3D, 3, "4..64(pow2)", 2, 1, True)]:
        text, _ = ref.csv_sweep(kind, m, nr, rho, T, analyze=an)
        for line in text.splitlines()[1:]:
            f = line.split(",")
            r = Fraction(int(f[9]), int(f[10]))
            assert rp.decimal_string(r) == f[11], line
            if an:
                assert rp.decimal_string(Fraction(int(f[12]), int(f[13]))) == f[14]
                assert rp.scheme_overhead_limit(api.map_kind[{"bb": "bb", "h3d": "h3d", "trapezoid": "h2d_trapezoid"}
                                                             [f[1]]], int(f[2])) == Fraction(int(f[12]), int(f[13]))
    assert rp.decimal_string(Fraction(-1, 3), 2) == "-0.33"
    assert rp.decimal_string(Fraction(1, 2), 0) == "1"


def test_text_report_lines():
    """text_report (report.hpp:483-511) on host rows (test_report.cpp:190-200)."""
    row = rp.measure_row(kind=api.map_kind.h2d, m=2, n=16, rho=1, blocks_launched=120, blocks_void=0,
                         threads_launched=120, threads_useful=120, overhead=Fraction(0), exact=True)
    text = rp.text_report([row], True)
    assert text == ("map=h2d m=2 n=16 rho=1 blocks=120 void=0 threads=120 useful=120 overhead=0 (0.000000)"
                    " Exact\n")
    bad = rp.measure_row(kind=api.map_kind.bb, m=3, n=4, blocks_launched=64, blocks_void=44, threads_launched=64,
                         threads_useful=20, overhead=Fraction(11, 5), witness=api.data_coord(2, 5, 1))
    assert rp.text_report([bad], True).endswith("overhead=11/5 (2.200000) NotExact witness=(2,5,1) mult=0\n")
    assert "Exact" not in rp.text_report([bad], False)
