"""HOPH statistics of Lemmas 1-3, exact rationals.

TEST INFRASTRUCTURE (like the rest of oracle/): the paper's aggregate statistics
of an (a:b) HOPH of l+1 groups, evaluated verbatim (SPEC
hoph_aggregate_matched / hoph_aggregate_empty).  They are not on the
scoring path: the comparison rules use the mass balance (R19) and the final
verdict the nominal-weight estimator (R21).

The lemmas model the layout as l+1 groups, "from l different one permutation
hashes": group j < l has k' bins, the last two groups both come from the
l-th hash.  Per the proof's convention the counts of those last two groups are
summed into N_l (`lemma_terms`).
"""
from __future__ import annotations

from fractions import Fraction


def lemma_terms(group_counts):
    """The lemmas' N_1 .. N_l from the l+1 per-group counts of a HOPH sketch pair
    (the last two groups summed)."""
    g = list(group_counts)
    if len(g) < 2:
        raise ValueError("the lemmas need l + 1 >= 2 groups")
    return g[:-2] + [g[-2] + g[-1]]


def hoph_aggregate(counts, r, l: int) -> Fraction:
    """Lemma 1 for matched bins, Lemma 2 for empty bins:
    N_h = (sum_{j=1}^{l-1} r^(2j) N_j + r^(2l-1) N_l) (l + 1), verbatim; counts = N_1..N_l."""
    r = Fraction(r)
    if len(counts) != l or l < 1:
        raise ValueError("counts must hold N_1 .. N_l")
    s = sum(r ** (2 * j) * Fraction(counts[j - 1]) for j in range(1, l))
    return (s + r ** (2 * l - 1) * Fraction(counts[l - 1])) * (l + 1)


def hoph_aggregate_probability(counts, r, l: int, kprime: int) -> Fraction:
    """The proof's first line with its k_j = k'/r^j: the probability that a bin of
    the k_h = (l+1) k' bins is matched (empty), sum_{j<l} r^j N_j / k_j + r^(l-1) N_l / k_l."""
    r = Fraction(r)
    kj = [Fraction(kprime) / r ** j for j in range(1, l + 1)]
    s = sum(r ** j * Fraction(counts[j - 1]) / kj[j - 1] for j in range(1, l))
    return s + r ** (l - 1) * Fraction(counts[l - 1]) / kj[l - 1]


def hoph_lemma3_estimate(n_mb, n_eb, r, l: int, kprime: int):
    """Lemma 3: R = sum_{j=1}^{l-1} r^j N_mb_j / (k_j - N_eb_j)
    + r^(l-1) N_mb_l / (k_l - N_eb_l).  k_j read as the bins the counts range over
    (R31): k' for j < l, 2 k' for the l-th term (the last two groups).
    A term with k_j - N_eb_j = 0 makes the estimate undefined (None)."""
    r = Fraction(r)
    est = Fraction(0)
    for j in range(1, l + 1):
        k = kprime if j < l else 2 * kprime
        den = k - n_eb[j - 1]
        if den <= 0:
            return None
        w = r ** j if j < l else r ** (l - 1)
        est += w * Fraction(n_mb[j - 1], den)
    return est
