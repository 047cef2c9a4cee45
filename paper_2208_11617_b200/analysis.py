"""The r/beta self-similar analysis (host-only, exact rationals), SURVEY 8(a)'s
last row: analysis.hpp:21-160 restated with Python Fractions.

The executable maps are the halving family (1/r, beta) = (2, 2) (maps.hpp,
SURVEY 0.4); this module predicts what other integral families would cover:
the orthotope-family volume V(S_n) = (n^m - beta^k) / ((1/r)^m - beta) for
n = (1/r)^k, its extra fraction alpha against the simplex, the covering onset
n0, and the ranked grid search behind BASELINE config C5's "r/beta sweep".
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction

from ._lib import InvalidArgument


def simplex_volume(n: int, m: int) -> int:
    """C(n+m-1, m): cells of the m-simplex of side n (core.hpp:105-114)."""
    return math.comb(n + m - 1, m) if n >= 1 else 0


@dataclass(frozen=True)
class self_similar_params:
    """analysis.hpp:21-33: 1/r >= beta > 1, m >= 1."""
    inv_r: int = 2
    beta: int = 2
    m: int = 2

    def __post_init__(self):
        if self.m < 1:
            raise InvalidArgument("self_similar_params: m must be >= 1")
        if self.beta <= 1:
            raise InvalidArgument("self_similar_params: beta must be > 1")
        if self.inv_r < self.beta:
            raise InvalidArgument("self_similar_params: 1/r must be >= beta")


@dataclass
class efficiency_report:
    """analysis.hpp:35-41"""
    volume_s: Fraction = Fraction(0)
    volume_simplex: int = 0
    alpha: Fraction = Fraction(0)
    n0: int = 0
    found: bool = False


def _exact_log(n: int, inv_r: int) -> int:
    if n < 1:
        raise InvalidArgument("self_similar_volume: n must be >= 1")
    k, v = 0, 1
    while v < n:
        v *= inv_r
        k += 1
    if v != n:
        raise InvalidArgument("self_similar_volume: n must be a power of 1/r")
    return k


def self_similar_volume(n: int, p: self_similar_params) -> Fraction:
    """V(S_n) for n = (1/r)^k: the recurrence V(n) = (n r)^m + beta V(n r),
    V(1) = 0, summed in closed form."""
    k = _exact_log(n, p.inv_r)
    ipow = p.inv_r ** p.m
    if ipow <= p.beta:
        raise InvalidArgument("self_similar_volume: (1/r)^m must exceed beta")
    return Fraction(n ** p.m - p.beta ** k, ipow - p.beta)


def extra_fraction_limit(m: int, p: self_similar_params | None = None) -> Fraction:
    """lim alpha for the halving family: m! / (2^m - 2) - 1."""
    if m < 2:
        raise InvalidArgument("extra_fraction_limit: m must be >= 2")
    p = p or self_similar_params(2, 2, m)
    if p.inv_r != 2 or p.beta != 2:
        raise InvalidArgument("extra_fraction_limit: defined for inv_r=2, beta=2")
    return Fraction(math.factorial(m), 2 ** m - 2) - 1


def extra_fraction_at(n: int, p: self_similar_params) -> Fraction:
    if n < 2:
        raise InvalidArgument("extra_fraction_at: n must be >= 2")
    return self_similar_volume(n, p) / simplex_volume(n - 1, p.m) - 1


def find_n0(p: self_similar_params, n_bound: int) -> efficiency_report:
    """The smallest power of 1/r (<= n_bound) whose family volume covers the simplex."""
    n = p.inv_r
    while n <= n_bound:
        vs = self_similar_volume(n, p)
        vd = simplex_volume(n - 1, p.m)
        if vs >= vd:
            return efficiency_report(vs, vd, vs / vd - 1, n, True)
        if n > n_bound // p.inv_r:
            break
        n *= p.inv_r
    return efficiency_report()


def optimize_params(m: int, inv_r_max: int, beta_max: int, n_eval: int):
    """Every integral 1/r >= beta > 1, ranked by |alpha| at the largest power of
    1/r <= n_eval, then smaller n0, smaller beta, smaller 1/r."""
    if n_eval < 2:
        raise InvalidArgument("optimize_params: n_eval must be >= 2")
    out = []
    for beta in range(2, beta_max + 1):
        for inv_r in range(beta, inv_r_max + 1):
            p = self_similar_params(inv_r, beta, m)
            n = inv_r
            while n <= n_eval // inv_r:
                n *= inv_r
            sweep = find_n0(p, n_eval)
            rep = efficiency_report(self_similar_volume(n, p), simplex_volume(n - 1, m), extra_fraction_at(n, p),
                                    sweep.n0, sweep.found)
            out.append((p, rep))
    if not out:
        raise InvalidArgument("optimize_params: empty feasible (1/r, beta) grid")
    big = 2 ** 63 - 1
    out.sort(key=lambda pr: (abs(pr[1].alpha), pr[1].n0 if pr[1].found else big, pr[0].beta, pr[0].inv_r))
    return out


def real_scaling_diagnostic(m: int, beta: int) -> tuple[float, float]:
    """(1/r, alpha_infinity) for the non-integral scaling (1/r)^m = m!."""
    if m < 2:
        raise InvalidArgument("real_scaling_diagnostic: m must be >= 2")
    if beta <= 1:
        raise InvalidArgument("real_scaling_diagnostic: beta must be > 1")
    mf = float(math.factorial(m))
    if beta >= mf:
        raise InvalidArgument("real_scaling_diagnostic: beta must be below m!")
    return mf ** (1.0 / m), beta / (mf - beta)


def csv_optimize(ranked, n_eval: int) -> str:
    """csv_optimize (report.hpp:448-472), schema slx-opt-1."""
    from .report import decimal_string
    out = "schema,m,inv_r,beta,n_eval,alpha_num,alpha_den,alpha_decimal,n0_found,n0\n"
    for p, rep in ranked:
        a = rep.alpha
        out += (f"slx-opt-1,{p.m},{p.inv_r},{p.beta},{n_eval},{a.numerator},{a.denominator},{decimal_string(a)},"
                f"{1 if rep.found else 0},{rep.n0 if rep.found else 0}\n")
    return out


def check_executable(p: self_similar_params | None) -> None:
    """The executable H maps are the (2, 2) family: any other
    (1/r, beta) is rejected on the 3-D path."""
    if p is not None and (p.inv_r, p.beta) != (2, 2):
        raise InvalidArgument("map_h3d: the executable map is the halving family (1/r, beta) = (2, 2)")
