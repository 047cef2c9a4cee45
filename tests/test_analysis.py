"""The r/beta analysis (SURVEY 8(a) last row; analysis.hpp) against the
reference: test_analysis.cpp's pinned values, and csv_optimize text
byte-identical to the reference's for the BASELINE C5 sweep grids."""
from fractions import Fraction

import pytest

from paper_2208_11617_b200 import analysis as A
from paper_2208_11617_b200 import api


def test_params_validation():
    A.self_similar_params(2, 2, 2)
    A.self_similar_params(5, 3, 4)
    for args in ((3, 1, 2), (2, 3, 2), (3, 2, 0)):
        with pytest.raises(api.InvalidArgument):
            A.self_similar_params(*args)


def test_volume_closed_form_and_recurrence():
    P = A.self_similar_params
    assert A.self_similar_volume(16, P(2, 2, 2)) == 120 == A.simplex_volume(15, 2)
    assert A.self_similar_volume(8, P(2, 2, 3)) == 84
    assert A.self_similar_volume(16, P(2, 2, 4)) == 4680
    assert A.self_similar_volume(1, P(2, 2, 2)) == 0
    with pytest.raises(api.InvalidArgument):
        A.self_similar_volume(12, P(2, 2, 2))
    with pytest.raises(api.InvalidArgument):
        A.self_similar_volume(2, P(2, 2, 1))
    for beta in range(2, 9):
        for inv_r in range(beta, 9):
            for m in range(2, 5):
                p = P(inv_r, beta, m)
                v, n = Fraction(0), 1
                for _ in range(1, 8):
                    prev = n ** m
                    n *= inv_r
                    v = prev + beta * v
                    assert A.self_similar_volume(n, p) == v


def test_limits_and_n0():
    P = A.self_similar_params
    assert [A.extra_fraction_limit(m) for m in (2, 3, 4, 5, 7)] == [0, 0, Fraction(5, 7), 3, 39]
    with pytest.raises(api.InvalidArgument):
        A.extra_fraction_limit(1)
    with pytest.raises(api.InvalidArgument):
        A.extra_fraction_limit(4, P(3, 2, 4))
    assert A.extra_fraction_at(8, P(2, 2, 3)) == 0 and A.extra_fraction_at(1024, P(2, 2, 2)) == 0
    r3 = A.find_n0(P(2, 2, 3), 1 << 12)
    assert r3.found and r3.n0 == 2 and r3.alpha == 0
    r5 = A.find_n0(P(2, 2, 5), 1 << 12)
    assert r5.found and r5.n0 == 2 and r5.volume_s == 1 and r5.volume_simplex == 1
    never = A.find_n0(P(8, 3, 2), 1 << 30)
    assert not never.found and never.n0 == 0
    top3 = A.optimize_params(3, 8, 8, 1 << 12)
    assert (top3[0][0].inv_r, top3[0][0].beta, top3[0][1].alpha) == (2, 2, 0)
    # for m = 3 only (2, 2) covers; (3, 3) gives alpha = -3/4
    assert all(r.alpha < 0 for p, r in top3[1:])
    assert dict(((p.inv_r, p.beta), r.alpha) for p, r in A.optimize_params(3, 8, 8, 2048))[(3, 3)] == Fraction(-3, 4)


def test_csv_optimize_byte_identical(ref):
    for m, ir, bm, ne in ((2, 8, 8, 4096), (3, 8, 8, 2048), (3, 8, 8, 256), (2, 2, 2, 4096), (4, 6, 5, 1000)):
        assert A.csv_optimize(A.optimize_params(m, ir, bm, ne), ne) == ref.csv_optimize(m, ir, bm, ne)


def test_executable_family_only():
    A.check_executable(None)
    A.check_executable(A.self_similar_params(2, 2, 3))
    with pytest.raises(api.InvalidArgument):
        A.check_executable(A.self_similar_params(3, 3, 3))
