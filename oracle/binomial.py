"""Exact binomial tails of Eq. 9-10 -- ORACLE, test infrastructure only.

X ~ Bin(K = k', p = T) is the number of matched bins in a K-bin comparison
part when the pair's similarity is exactly T ("X ~ F(T, K)"; read as
trials = k', success probability = T, R8, pinned by Table 2,
P:396-420).  The two branches of Eq. 10 are read as (R9)

    lower(m) = P(X <= m)   ("F(x < X)" column of Table 2 at X = m + 1)
    upper(m) = P(X >= m)   ("F(x >= X)" column of Table 2 at X = m)

Everything is an exact rational (fractions.Fraction); T is a rational
t_num/t_den and eps enters as the exact value of the given float.  The
small-probability test of Definition 1 is `tail <= eps` (R13).
"""
from __future__ import annotations

from fractions import Fraction
from functools import lru_cache
from math import comb


@lru_cache(maxsize=None)
def pmf(K: int, t_num: int, t_den: int) -> tuple:
    """P(X = j), j = 0..K, exactly."""
    T = Fraction(t_num, t_den)
    return tuple(comb(K, j) * T ** j * (1 - T) ** (K - j) for j in range(K + 1))


def lower_tail(m: int, K: int, t_num: int, t_den: int) -> Fraction:
    """P(X <= m); m may be -1 (-> 0)."""
    if m < -1 or m > K:
        raise ValueError("lower_tail: m out of [-1, K]")
    return sum(pmf(K, t_num, t_den)[: m + 1], Fraction(0))


def upper_tail(m: int, K: int, t_num: int, t_den: int) -> Fraction:
    """P(X >= m); m may be K+1 (-> 0)."""
    if m < 0 or m > K + 1:
        raise ValueError("upper_tail: m out of [0, K+1]")
    return sum(pmf(K, t_num, t_den)[m:], Fraction(0))


@lru_cache(maxsize=None)
def small_probability_tables(K: int, t_num: int, t_den: int, eps: float):
    """Definition 1 evaluated at every integer point:
    lower_le[m] = (P(X <= m) <= eps) for m in 0..K,
    upper_le[m] = (P(X >= m) <= eps) for m in 0..K+1."""
    e = Fraction(eps)
    lower_le = bytes(int(lower_tail(m, K, t_num, t_den) <= e) for m in range(K + 1))
    upper_le = bytes(int(upper_tail(m, K, t_num, t_den) <= e) for m in range(K + 2))
    return lower_le, upper_le
