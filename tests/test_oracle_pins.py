"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test names the passage it pins (P:n = PAPER.md line n, S:n = SPEC.md
line n, Rn = DESIGN.md reading n).  The oracle is never compared with
itself: the expected values are the paper's printed numbers (tests/golden/),
closed forms, brute force on tiny inputs, or statistical invariants.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import EMPTY, binomial
from workloads import make_csr

E = EMPTY


def _sk(lst):
    return [E if v is None else v for v in lst]


# --------------------------------------------------------------------- Eq. 10 / Table 2
def test_table2_binomial_tails(golden):
    """Table 2: all 20 printed rows, both columns (R8, R9)."""
    g = golden("table2.json")
    K, tn, td = g["K"], g["t_num"], g["t_den"]
    for X, lo_printed, up_printed in g["rows"]:
        lo = float(binomial.lower_tail(X - 1, K, tn, td))  # F(x < X)
        up = float(binomial.upper_tail(X, K, tn, td))      # F(x >= X)
        assert lo == pytest.approx(lo_printed, rel=1e-5), X
        assert up == pytest.approx(up_printed, rel=1e-5), X


def test_binomial_complement_and_monotone():
    """lower(m) + upper(m+1) = 1 exactly; monotone; ends."""
    for K, tn, td in [(16, 7, 10), (32, 4, 5), (100, 3, 5), (5, 1, 2)]:
        lo = [binomial.lower_tail(m, K, tn, td) for m in range(-1, K + 1)]
        up = [binomial.upper_tail(m, K, tn, td) for m in range(0, K + 2)]
        for m in range(0, K + 1):
            assert binomial.lower_tail(m, K, tn, td) + binomial.upper_tail(m + 1, K, tn, td) == 1
        assert all(a <= b for a, b in zip(lo, lo[1:]))
        assert all(a >= b for a, b in zip(up, up[1:]))
        assert lo[0] == 0 and lo[-1] == 1 and up[0] == 1 and up[-1] == 0


def test_binomial_brute_force_small():
    """Brute force: enumerate all 2^K outcomes of K Bernoulli(T) trials."""
    K, T = 8, Fraction(3, 10)
    import itertools
    dist = [Fraction(0)] * (K + 1)
    for bits in itertools.product([0, 1], repeat=K):
        p = Fraction(1)
        for b in bits:
            p *= T if b else 1 - T
        dist[sum(bits)] += p
    for m in range(K + 1):
        assert binomial.lower_tail(m, K, 3, 10) == sum(dist[: m + 1])
        assert binomial.upper_tail(m, K, 3, 10) == sum(dist[m:])


# --------------------------------------------------------------------- O1 psi
@pytest.mark.parametrize("V", [1, 2, 3, 17, 1000, 65536, 1 << 20, 1000003])
def test_psi_is_a_bijection(V):
    """S:33 'mapping is a bijection'; exhaustive over [0, V)."""
    for seed in (0, 1, 0xDEADBEEF):
        img = oracle.psi(np.arange(V, dtype=np.uint64), V, seed)
        assert img.max(initial=0) < V
        assert len(np.unique(img)) == V


def test_psi_2_32_injective_on_sample():
    """|V| = 2^32: no collision among 2^20 consecutive ids plus 2^20 random ids
    (a random non-injective map would show ~500 birthday collisions)."""
    rng = np.random.default_rng(7)
    x = np.unique(np.concatenate([np.arange(1 << 20, dtype=np.uint64),
                                  rng.integers(0, 1 << 32, size=1 << 20, dtype=np.uint64)]))
    img = oracle.psi(x, 1 << 32, 12345)
    assert img.max() < (1 << 32)
    assert len(np.unique(img)) == len(x)


def test_psi_identity_and_determinism():
    """S:113 identity constructor; S:34 same seed + size => same mapping."""
    x = np.arange(17, dtype=np.uint64)
    assert (oracle.psi(x, 17, 5, identity=True) == x).all()
    a = oracle.psi(np.arange(1000, dtype=np.uint64), 1 << 32, 42)
    b = oracle.psi(np.arange(1000, dtype=np.uint64), 1 << 32, 42)
    c = oracle.psi(np.arange(1000, dtype=np.uint64), 1 << 32, 43)
    assert (a == b).all() and not (a == c).all()


# --------------------------------------------------------------------- O2 / O3 OPH sketch
def test_flat_layout_floor_rule_brute_force():
    """S:38 bin i covers [floor(i|V|/k), floor((i+1)|V|/k)); S:107 |V|=17,k=4
    gives boundaries 0,4,8,12,17.  Single-element sets under the identity
    permutation expose (bin, offset) of every p."""
    for V, k in [(17, 4), (100, 7), (64, 64), (1000, 3), (5, 5)]:
        offs, ids = make_csr([[p] for p in range(V)])
        F = oracle.oph_sketch(offs, ids, V, k, 0, identity=True)
        starts = [b * V // k for b in range(k + 1)]
        for p in range(V):
            b = max(i for i in range(k) if starts[i] <= p)
            row = F[p]
            assert row[b] == p - starts[b]
            assert all(row[j] == E for j in range(k) if j != b)
    assert [b * 17 // 4 for b in range(5)] == [0, 4, 8, 12, 17]


def test_oph_worked_example(golden):
    """P:158-160 sketches [1,1,2,0], [1,2,2,0], [2,(x),1,0]; estimates 0.75 and
    0.333 (EitherEmpty), 1/4 under JointEmpty (Eq. 4); exact J 0.5, 0.375."""
    g = golden("oph_example.json")
    names = ["D1", "D2", "D3"]
    offs, ids = make_csr([g["sets"][n] for n in names])
    F = oracle.oph_sketch(offs, ids, g["vocab_size"], g["k"], 0, identity=True)
    for i, n in enumerate(names):
        assert list(F[i]) == _sk(g["sketch"][n])
    either = oracle.compare_full(F, F, t_num=7, t_den=10, joint=False)
    joint = oracle.compare_full(F, F, t_num=7, t_den=10, joint=True)
    assert either[0, 1]["n_mb"] == 3 and either[0, 1]["estimate"] == 0.75 and joint[0, 1]["estimate"] == 0.75
    assert either[0, 2]["n_mb"] == 1
    assert either[0, 2]["estimate"] == pytest.approx(1 / 3, abs=1e-15)
    assert joint[0, 2]["estimate"] == 0.25
    for p in g["pairs"]:
        a, b = g["sets"][p["a"]], g["sets"][p["b"]]
        j, _, _ = oracle.jaccard(a, b)
        assert j == p["jaccard"]


def test_oph_empty_set_sketch():
    """S:210 empty FeatureSet -> all (x); S:251 two all-(x) sketches -> undefined."""
    offs, ids = make_csr([[], [3]])
    F = oracle.oph_sketch(offs, ids, 16, 4, 9)
    assert (F[0] == E).all()
    r = oracle.compare_full(F[:1], F[:1], t_num=1, t_den=2)
    assert r[0, 0]["flags"] & oracle.UNDEFINED and r[0, 0]["verdict"] == 0


# --------------------------------------------------------------------- O4 / O5 HOPH
def test_hoph_layout_worked_example(golden):
    """(|V|=17, 1:1, k'=2) -> [0,8), [8,12), [12,17) (R17, R18)."""
    g = golden("hoph_example.json")
    assert oracle.hoph_layout(g["vocab_size"], g["a"], g["b"], g["kprime"]) == [tuple(x) for x in g["layout"]]


@pytest.mark.parametrize("V,kp,L", [(1 << 16, 16, 12), (1 << 16, 32, 11), (1 << 20, 32, 15),
                                    (1 << 32, 32, 27), (1 << 16, 100, 10)])
def test_hoph_layout_group_counts(V, kp, L):
    """Recursive 1:1 split: group j has length floor(R/2) of the
    remainder R until a half would be <= k'.  For |V| = 2^m the closed form is
    lengths 2^(m-1), 2^(m-2), ..., then the last remainder."""
    lay = oracle.hoph_layout(V, 1, 1, kp)
    assert len(lay) == L
    assert lay[0] == (0, V // 2)
    assert sum(length for _, length in lay) == V
    assert all(s2 == s1 + l1 for (s1, l1), (s2, _) in zip(lay, lay[1:]))
    assert all(length >= kp for _, length in lay)


def test_hoph_layout_properties_random():
    """S:401 group lengths >= k' and sum to |V|; S:400 |V| = 4k' -> two groups."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        kp = int(rng.integers(1, 50))
        V = int(rng.integers(2 * kp, 10 ** 6))
        a, b = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        lay = oracle.hoph_layout(V, a, b, kp)
        assert sum(length for _, length in lay) == V and all(length >= kp for _, length in lay)
        for (s, length), (s2, _) in zip(lay, lay[1:]):  # every non-final group is floor(a R/(a+b))
            R = V - s
            assert length == a * R // (a + b)
    assert oracle.hoph_layout(4 * 8, 1, 1, 8) == [(0, 16), (16, 16)]


def test_hoph_worked_example(golden):
    """sketches [[1,1],[(x),0],[0,1]], [[1,2],[(x),0],[0,0]]; D3 from the
    raw sample at P:478; estimates 0.625 and 0.375 with nominal weights (R21)."""
    g = golden("hoph_example.json")
    og = golden("oph_example.json")
    names = ["D1", "D2", "D3"]
    offs, ids = make_csr([og["sets"][n] for n in names])
    H = oracle.hoph_sketch(offs, ids, g["vocab_size"], g["layout"], g["kprime"], 0, identity=True)
    for i, n in enumerate(names):
        assert list(H[i]) == _sk(g["sketch"][n])
    for p in g["pairs"]:
        a, b = names.index(p["a"]), names.index(p["b"])
        r = oracle.hoph_estimate(H[a], H[b], L=3, kprime=2, a=1, b=1, t_num=1, t_den=2)
        assert r["estimate"] == p["estimate_num"] / p["estimate_den"]


def test_hoph_weights_nominal():
    """Lemma 3 with l = L: w_j = r(1-r)^(j-1), w_L = (1-r)^(L-1).  They
    sum to 1 and at 1:1 on |V| = 2^m equal the group shares len_j/|V|."""
    for a, b, L in [(1, 1, 27), (1, 2, 10), (2, 1, 18), (3, 5, 7), (1, 1, 1)]:
        c, D = oracle.hoph_weights(a, b, L)
        r = Fraction(a, a + b)
        want = [r * (1 - r) ** (j - 1) for j in range(1, L)] + [(1 - r) ** (L - 1)]
        assert [Fraction(x, D) for x in c] == want
        assert sum(c) == D
    lay = oracle.hoph_layout(1 << 32, 1, 1, 32)
    c, D = oracle.hoph_weights(1, 1, len(lay))
    assert [Fraction(x, D) for x in c] == [Fraction(length, 1 << 32) for _, length in lay]


def test_hoph_single_group_reduces_to_oph():
    """|V| = 2k' gives one group; the HOPH estimator is then the OPH estimator
    of that group's k' bins (Eq. 6)."""
    rng = np.random.default_rng(11)
    V, kp = 64, 32
    lay = oracle.hoph_layout(V, 1, 1, kp)
    assert lay == [(0, 64)]
    sets = [sorted(rng.choice(V, size=int(rng.integers(0, 40)), replace=False).tolist()) for _ in range(30)]
    offs, ids = make_csr(sets)
    H = oracle.hoph_sketch(offs, ids, V, lay, kp, 77)
    F = oracle.oph_sketch(offs, ids, V, kp, 77)
    assert (H == F).all()
    full = oracle.compare_full(F, F, t_num=1, t_den=2)
    for i in range(30):
        for j in range(30):
            h = oracle.hoph_estimate(H[i], H[j], L=1, kprime=kp, a=1, b=1, t_num=1, t_den=2)
            assert h["flags"] == full[i, j]["flags"]
            if not h["flags"]:
                assert h["estimate"] == pytest.approx(full[i, j]["estimate"], abs=1e-15)
                assert h["verdict"] == full[i, j]["verdict"]


# --------------------------------------------------------------------- O9 GOPH
def _goph_pair(matches, kp, n):
    """Two flat sketches whose group l has exactly matches[l] matched bins and
    no empty bin."""
    q = np.zeros((1, n * kp), dtype=np.uint32)
    s = np.ones((1, n * kp), dtype=np.uint32)
    for l, m in enumerate(matches):
        s[0, l * kp: l * kp + m] = 0
    return q, s


def test_goph_example1(golden):
    """Example 1: M_ra 59.4, 66.25, 74.28, 85 and NotSimilar after
    group 4, F(x >= 85) = 5.0732e-8 (R10, R11, R12)."""
    g = golden("example1.json")
    q, s = _goph_pair(g["matches"] + [0] * 6, g["kprime"], g["n"])
    r, tr = oracle.compare_goph(q, s, n=g["n"], kprime=g["kprime"], t_num=g["t_num"], t_den=g["t_den"],
                                eps=g["eps"], trace=True)
    assert r[0, 0]["groups"] == g["groups_compared"] and r[0, 0]["verdict"] == 0
    assert r[0, 0]["flags"] == oracle.EARLY
    for l, (printed, tol) in enumerate(g["m_ra_printed"]):
        m_ra = tr[0, 0, l, 0] / tr[0, 0, l, 1]
        assert abs(m_ra - printed) <= tol + 1e-12, (l, m_ra)
    assert float(binomial.upper_tail(85, 100, 3, 5)) == pytest.approx(g["upper_85"], rel=1e-5)


# ---- O9e empty-aware GOPH (E1-E4)
def test_goph_e_example1_without_empties(golden):
    """E2 reduces to Alg. 1 when no bin is excluded: Example 1 gives
    the same M_ra 59.4, 66.25, 74.28, 85 and NotSimilar after group 4."""
    g = golden("example1.json")
    q, s = _goph_pair(g["matches"] + [0] * 6, g["kprime"], g["n"])
    r, tr = oracle.compare_goph(q, s, n=g["n"], kprime=g["kprime"], t_num=g["t_num"], t_den=g["t_den"],
                                eps=g["eps"], trace=True, empty_aware=True)
    assert (r[0, 0]["groups"], r[0, 0]["verdict"], r[0, 0]["flags"]) == (g["groups_compared"], 0, oracle.EARLY)
    for l, (printed, tol) in enumerate(g["m_ra_printed"]):
        assert abs(tr[0, 0, l, 0] / tr[0, 0, l, 1] - printed) <= tol + 1e-12


def test_goph_e_example1_excluded_tail(golden):
    """Example 1's counts (65, 5 matched of 100 in groups 1-2) with every bin of
    groups 5-10 empty on the set side (EitherEmpty): D = 400 trials.  Group 1:
    R = 300, M_ra = 100 (0.6*400 - 65)/300 = 58.33 < 60, P(X <= 58) = 0.38 > eps:
    continue.  Group 2: R = 200, M_ra = 100 (240 - 70)/200 = 85 >= 60 and
    P(X >= 85) = 5.0732e-8 <= eps (the paper's printed tail): NotSimilar
    after 2 groups -- Alg. 1 itself needs 4 (M_ra 66.25 at group 2)."""
    g = golden("example1.json")
    kp, n = g["kprime"], g["n"]
    q, s = _goph_pair(g["matches"] + [0] * 6, kp, n)
    s[0, 4 * kp:] = oracle.EMPTY
    r, tr = oracle.compare_goph(q, s, n=n, kprime=kp, t_num=g["t_num"], t_den=g["t_den"], eps=g["eps"],
                                trace=True, empty_aware=True)
    assert Fraction(int(tr[0, 0, 0, 0]), int(tr[0, 0, 0, 1])) == Fraction(175, 3)
    assert Fraction(int(tr[0, 0, 1, 0]), int(tr[0, 0, 1, 1])) == 85
    assert float(binomial.upper_tail(85, 100, 3, 5)) == pytest.approx(g["upper_85"], rel=1e-5)
    assert (r[0, 0]["groups"], r[0, 0]["verdict"], r[0, 0]["flags"]) == (2, 0, oracle.EARLY)
    assert (r[0, 0]["n_mb"], r[0, 0]["n_excl"]) == (70, 0)
    r0 = oracle.compare_goph(q, s, n=n, kprime=kp, t_num=g["t_num"], t_den=g["t_den"], eps=g["eps"])
    assert r0[0, 0]["groups"] == 4


def test_goph_e_reduces_to_alg1_without_empties():
    """No excluded bin: the variant's records and M_ra traces equal Alg. 1's
    (E2) on random per-group match counts, four parameter sets."""
    rng = np.random.default_rng(55)
    for kp, n, tn, td, eps in [(16, 4, 7, 10, 1e-4), (32, 8, 7, 10, 1e-4), (32, 8, 4, 5, 1e-3), (10, 6, 1, 2, 1e-2)]:
        Q, S = [], []
        for _ in range(200):
            q, s = _goph_pair(rng.binomial(kp, rng.uniform(0, 1), size=n).tolist(), kp, n)
            Q.append(q[0]); S.append(s[0])
        Q, S = np.array(Q), np.array(S)
        for joint in (False, True):
            kw = dict(n=n, kprime=kp, t_num=tn, t_den=td, eps=eps, joint=joint, trace=True)
            a, ta = oracle.compare_goph(Q, S, **kw)
            b, tb = oracle.compare_goph(Q, S, empty_aware=True, **kw)
            assert np.array_equal(a, b)
            d = np.arange(len(Q))
            # per stop level, the traced M_ra agree as rationals (the variant's are scaled by k')
            for l in range(n - 1):
                live = a["groups"][d, d] > l
                assert np.array_equal(ta[d, d, l, 0][live] * tb[d, d, l, 1][live],
                                      tb[d, d, l, 0][live] * ta[d, d, l, 1][live])


def test_goph_e_final_and_complete_are_full_oph():
    """E3: a pair the variant does not stop early (flags without EARLY) carries
    the full-OPH record (Eq. 6) -- at the last group, or earlier when every
    remaining bin is excluded; both empty modes, random sketches with empties."""
    rng = np.random.default_rng(56)
    n, kp = 8, 16
    Q = rng.integers(0, 2, size=(40, n * kp)).astype(np.uint32)
    S = rng.integers(0, 2, size=(60, n * kp)).astype(np.uint32)
    Q[rng.random(Q.shape) < 0.3] = oracle.EMPTY
    S[rng.random(S.shape) < 0.3] = oracle.EMPTY
    S[:20, 5 * kp:] = oracle.EMPTY            # groups 6-8 empty on the set side
    Q[:10, 3 * kp:] = oracle.EMPTY            # groups 4-8 empty on the query side
    for joint in (False, True):
        full = oracle.compare_full(Q, S, t_num=1, t_den=2, joint=joint)
        e = oracle.compare_goph(Q, S, n=n, kprime=kp, t_num=1, t_den=2, eps=1e-3, joint=joint, empty_aware=True)
        done = (e["flags"] & oracle.EARLY) == 0
        assert done.any() and (~done).any()
        for f in ("n_mb", "n_excl", "verdict", "flags"):
            assert np.array_equal(e[f][done], full[f][done]), f
        assert np.array_equal(e["estimate"][done], full["estimate"][done])
        if not joint:  # EitherEmpty: queries 0-9 x sets 0-19 have no trial past group 3
            assert (e["groups"][:10, :20] <= 3).all()
            assert done[:10, :20].any()


def test_goph_degenerate_traces():
    """S:347-348 (A.2): identical sketches -> Similar at the first l where
    lower(floor((600-100l)/(10-l))) <= 1e-4 (= group 4); zero matches ->
    NotSimilar at the first l where M_ra > 100 or upper(ceil(600/(10-l))) <= 1e-4
    (= group 3).  k'=100, n=10, T=0.6."""
    def first_stop_identical():
        for l in range(1, 10):
            m = Fraction(600 - 100 * l, 10 - l)
            if m <= 0 or binomial.lower_tail(int(m), 100, 3, 5) <= Fraction(1e-4):
                return l

    def first_stop_zero():
        for l in range(1, 10):
            m = Fraction(600, 10 - l)
            if m > 100 or binomial.upper_tail(-(-m.numerator // m.denominator), 100, 3, 5) <= Fraction(1e-4):
                return l
    assert first_stop_identical() == 4 and first_stop_zero() == 3
    q, s = _goph_pair([100] * 10, 100, 10)
    r = oracle.compare_goph(q, s, n=10, kprime=100, t_num=3, t_den=5, eps=1e-4)
    assert (r[0, 0]["groups"], r[0, 0]["verdict"]) == (4, 1)
    q, s = _goph_pair([0] * 10, 100, 10)
    r = oracle.compare_goph(q, s, n=10, kprime=100, t_num=3, t_den=5, eps=1e-4)
    assert (r[0, 0]["groups"], r[0, 0]["verdict"]) == (3, 0)


def test_goph_exact_rational_cross_check():
    """Algorithm 1 re-evaluated with Fractions in the paper's own (unscaled)
    form on random per-group match counts: same stop group and verdict as the
    oracle's scaled-integer evaluation (guards R16, floors/ceils R12)."""
    rng = np.random.default_rng(5)
    for kp, n, tn, td, eps in [(16, 4, 7, 10, 1e-4), (32, 8, 7, 10, 1e-4), (32, 8, 4, 5, 1e-3), (10, 6, 1, 2, 1e-2)]:
        T = Fraction(tn, td)
        lo, up = binomial.small_probability_tables(kp, tn, td, eps)
        for _ in range(300):
            p = rng.uniform(0, 1)
            matches = rng.binomial(kp, p, size=n).tolist()
            q, s = _goph_pair(matches, kp, n)
            r = oracle.compare_goph(q, s, n=n, kprime=kp, t_num=tn, t_den=td, eps=eps)[0, 0]
            Mc, want = 0, None
            for l in range(1, n + 1):
                Mc += matches[l - 1]
                if l == n:
                    want = (n, int(Fraction(Mc, n * kp) >= T))
                    break
                Mra = (n * kp * T - Mc) / (n - l)
                if Mra <= 0:
                    want = (l, 1)
                elif Mra > kp:
                    want = (l, 0)
                elif Mra < kp * T and lo[int(Mra)]:
                    want = (l, 1)
                elif Mra >= kp * T and up[-(-Mra.numerator // Mra.denominator)]:
                    want = (l, 0)
                if want:
                    break
            assert (r["groups"], r["verdict"]) == want


# --------------------------------------------------------------------- O10 HOPH filter
def test_hoph_example2(golden):
    """Example 2: 40 matches in group 1 of a 1:1 layout -> P_r = 0.8,
    P_r k' = 80, F(x >= 80) = 1.64119e-5 <= eps -> NotSimilar after 1 group."""
    g = golden("example2.json")
    lay = oracle.hoph_layout(g["vocab_size"], g["a"], g["b"], g["kprime"])
    L, kp = len(lay), g["kprime"]
    q = np.zeros((1, L * kp), dtype=np.uint32)
    s = np.ones((1, L * kp), dtype=np.uint32)
    s[0, :g["first_group_matches"]] = 0
    r, tr = oracle.compare_hoph(q, s, L=L, kprime=kp, a=1, b=1, t_num=g["t_num"], t_den=g["t_den"],
                                eps=g["eps"], trace=True)
    num, den = tr[0, 0, 0]
    assert Fraction(int(num), int(den)) == g["x"]
    assert (r[0, 0]["groups"], r[0, 0]["verdict"]) == (g["groups_compared"], 0)
    assert float(binomial.upper_tail(80, 100, 3, 5)) == pytest.approx(g["upper_80"], rel=1e-5)


def test_hoph_e_example2(golden):
    """The empty-aware HOPH rule (EH1-EH5) has no excluded bin in Example 2 and
    reproduces it: x = 80 as a rational, NotSimilar after group 1."""
    g = golden("example2.json")
    lay = oracle.hoph_layout(g["vocab_size"], g["a"], g["b"], g["kprime"])
    L, kp = len(lay), g["kprime"]
    q = np.zeros((1, L * kp), dtype=np.uint32)
    s = np.ones((1, L * kp), dtype=np.uint32)
    s[0, :g["first_group_matches"]] = 0
    r, tr = oracle.compare_hoph(q, s, L=L, kprime=kp, a=1, b=1, t_num=g["t_num"], t_den=g["t_den"],
                                eps=g["eps"], trace=True, empty_aware=True)
    num, den = tr[0, 0, 0]
    assert Fraction(int(num), int(den)) == g["x"]
    assert (r[0, 0]["groups"], r[0, 0]["verdict"]) == (g["groups_compared"], 0)


def _hoph_pair_groups(M, ex, kp):
    """A HOPH sketch pair whose group j has M[j] matched bins and ex[j] bins empty on
    both sides (excluded in either mode), the rest unequal and non-empty."""
    L = len(M)
    q = np.zeros(L * kp, dtype=np.uint32)
    s = np.ones(L * kp, dtype=np.uint32)
    for j in range(L):
        s[j * kp: j * kp + M[j]] = 0
        q[j * kp + kp - ex[j]: (j + 1) * kp] = E
        s[j * kp + kp - ex[j]: (j + 1) * kp] = E
    return q, s


def test_hoph_e_excluded_group_hand_example():
    """EH2-EH3 by hand: k' = 4, L = 3 (1:1: c = [2, 1, 1], D = 4), T = 1/2, group 2 fully
    excluded, so C_K = 3 and after group 1 the usable weight left is W_1 = c_3 = 1.
      m_1 = 3 of 4: A_1 = 2 * 3/4 = 3/2, x = k' (T C_K - A_1) / W_1 = 4 (3/2 - 3/2) = 0
                    -> Similar at group 1;  Alg. 2: S_1 = 6, x = (T D k' - S_1) / W_1' =
                    (8 - 6) / 2 = 1, P(X <= 1) = 5/16 > eps -> it continues.
      m_1 = 0:      x = 4 * 3/2 / 1 = 6 > k' -> NotSimilar at group 1;  Alg. 2: x = 8 / 2 = 4,
                    P(X >= 4) = 1/16 > eps -> it continues."""
    kp = 4
    for m1, verdict, x in [(3, 1, Fraction(0)), (0, 0, Fraction(6))]:
        q, s = _hoph_pair_groups([m1, 0, 0], [0, kp, 0], kp)
        kw = dict(L=3, kprime=kp, a=1, b=1, t_num=1, t_den=2, eps=1e-3, trace=True)
        r, tr = oracle.compare_hoph(q[None], s[None], empty_aware=True, **kw)
        num, den = tr[0, 0, 0]
        assert Fraction(int(num), int(den)) == x
        assert (r[0, 0]["groups"], r[0, 0]["verdict"], r[0, 0]["flags"]) == (1, verdict, oracle.EARLY)
        p = oracle.compare_hoph(q[None], s[None], **kw)[0][0, 0]
        assert p["groups"] > 1


def test_hoph_e_reduces_to_alg2_without_empties():
    """No excluded bin: the variant's records equal Algorithm 2's (R19) on random per-group
    match counts (1:1 and 1:2 layouts, three parameter sets, both empty modes)."""
    rng = np.random.default_rng(66)
    for kp, L, a, b, tn, td, eps in [(16, 6, 1, 1, 7, 10, 1e-4), (32, 8, 1, 1, 4, 5, 1e-3), (10, 5, 1, 2, 1, 2, 1e-2)]:
        Q, S = [], []
        for _ in range(200):
            q, s = _hoph_pair_groups(rng.binomial(kp, rng.uniform(0, 1), size=L).tolist(), [0] * L, kp)
            Q.append(q); S.append(s)
        Q, S = np.array(Q), np.array(S)
        for joint in (False, True):
            kw = dict(L=L, kprime=kp, a=a, b=b, t_num=tn, t_den=td, eps=eps, joint=joint)
            assert np.array_equal(oracle.compare_hoph(Q, S, **kw), oracle.compare_hoph(Q, S, empty_aware=True, **kw))


def test_hoph_e_final_records_are_the_estimator():
    """EH4 / EH5: a pair the variant does not stop early carries the HOPH estimator's record
    over all groups (R21, R22); a pair with no matched bin is never Similar."""
    rng = np.random.default_rng(67)
    kp, L = 8, 5
    Q, S = [], []
    for _ in range(400):
        ex = [int(x) if rng.random() < 0.6 else kp for x in rng.integers(0, kp, size=L)]
        M = [int(rng.integers(0, kp - e + 1)) for e in ex]
        q, s = _hoph_pair_groups(M, ex, kp)
        Q.append(q); S.append(s)
    Q, S = np.array(Q), np.array(S)
    for joint in (False, True):
        r = oracle.compare_hoph(Q, S, L=L, kprime=kp, a=1, b=1, t_num=3, t_den=5, eps=1e-3, joint=joint,
                                empty_aware=True)
        d = np.arange(len(Q))
        rr = r[d, d]
        done = (rr["flags"] & oracle.EARLY) == 0
        assert done.sum() > 50 and (~done).sum() > 50
        for i in np.nonzero(done)[0]:
            h = oracle.hoph_estimate(Q[i], S[i], L=L, kprime=kp, a=1, b=1, t_num=3, t_den=5, joint=joint)
            assert (rr["verdict"][i], rr["flags"][i], rr["n_mb"][i], rr["n_excl"][i]) == \
                (h["verdict"], h["flags"], h["n_mb"], h["n_excl"])
            assert rr["estimate"][i] == h["estimate"]
        nomatch = np.array([((Q[i] == S[i]) & (Q[i] != E)).sum() == 0 for i in range(len(Q))])
        assert nomatch.any() and (rr["verdict"][nomatch] == 0).all()


def test_hoph_mass_balance_cross_check():
    """Algorithm 2 with the mass balance P_r = (T - sum_{j<=l} w_j M_j/k') /
    sum_{j>l} w_j (R19) re-evaluated with Fractions on random match counts."""
    rng = np.random.default_rng(9)
    for kp, L, a, b, tn, td, eps in [(16, 12, 1, 1, 7, 10, 1e-4), (32, 10, 1, 2, 4, 5, 1e-4), (8, 6, 2, 1, 1, 2, 1e-2)]:
        T = Fraction(tn, td)
        r_ = Fraction(a, a + b)
        w = [r_ * (1 - r_) ** (j - 1) for j in range(1, L)] + [(1 - r_) ** (L - 1)]
        lo, up = binomial.small_probability_tables(kp, tn, td, eps)
        for _ in range(300):
            p = rng.uniform(0, 1)
            matches = rng.binomial(kp, p, size=L).tolist()
            q = np.zeros((1, L * kp), dtype=np.uint32)
            s = np.ones((1, L * kp), dtype=np.uint32)
            for l, m in enumerate(matches):
                s[0, l * kp: l * kp + m] = 0
            r = oracle.compare_hoph(q, s, L=L, kprime=kp, a=a, b=b, t_num=tn, t_den=td, eps=eps)[0, 0]
            want = None
            for l in range(1, L + 1):
                if l == L:
                    est = sum(w[j] * Fraction(matches[j], kp) for j in range(L))
                    want = (L, int(est >= T))
                    break
                Pr = (T - sum(w[j] * Fraction(matches[j], kp) for j in range(l))) / sum(w[l:])
                x = Pr * kp
                if x <= 0:
                    want = (l, 1)
                elif x > kp:
                    want = (l, 0)
                elif Pr < T and lo[int(x)]:
                    want = (l, 1)
                elif Pr >= T and up[-(-x.numerator // x.denominator)]:
                    want = (l, 0)
                if want:
                    break
            assert (r["groups"], r["verdict"]) == want


# --------------------------------------------------------------------- estimators: unbiasedness (Eq. 7)
def _pair_with_union(g, J, V, rng):
    inter = int(round(J * g))
    a_only = (g - inter) // 2
    b_only = g - inter - a_only
    u = rng.choice(V, size=g, replace=False)
    A = np.sort(u[: inter + a_only])
    B = np.sort(np.concatenate([u[:inter], u[inter + a_only:]]))
    return A, B, Fraction(inter, g)


@pytest.mark.parametrize("J", [0.25, 0.5, 0.8])
def test_oph_unbiased_joint_empty(J):
    """Eq. 7: over 10^4 permutations, g = 4096, k = 256,
    the mean JointEmpty OPH estimate is within 3 standard errors of J."""
    rng = np.random.default_rng(int(J * 100))
    V, k = 1 << 16, 256
    A, B, Jt = _pair_with_union(4096, J, V, rng)
    offs, ids = make_csr([A, B])
    ests = []
    for seed in range(10_000):
        F = oracle.oph_sketch(offs, ids, V, k, seed)
        r = oracle.compare_full(F[:1], F[1:], t_num=1, t_den=2, joint=True)[0, 0]
        ests.append(r["estimate"])
    ests = np.array(ests)
    se = ests.std(ddof=1) / np.sqrt(len(ests))
    assert abs(ests.mean() - float(Jt)) < 3 * se


def test_oph_variance_eq8():
    """Eq. 8 (Li-Owen-Zhang's OPH variance): for the JointEmpty
    estimator with g = |D1 u D2| and N_eb jointly empty bins,
    var = R(1-R)(E[1/(k - N_eb)](1 + 1/(g-1)) - 1/(g-1)).  g = 100 over k = 64
    bins leaves ~13 jointly empty bins per permutation, so the E[.] term is far
    from 1/k; over 6000 permutations the sample variance is within 10 % of the
    formula (its own standard error is ~2 %), while the 1/k form (empty bins
    ignored) misses by more than 15 %."""
    rng = np.random.default_rng(41)
    V, k, g = 1 << 16, 64, 100
    A, B, Jt = _pair_with_union(g, 0.4, V, rng)
    offs, ids = make_csr([A, B])
    ests, inv = [], []
    for seed in range(6000):
        F = oracle.oph_sketch(offs, ids, V, k, seed)
        r = oracle.compare_full(F[:1], F[1:], t_num=1, t_den=2, joint=True)[0, 0]
        ests.append(r["estimate"])
        inv.append(1.0 / (k - int(r["n_excl"])))
    ests = np.array(ests)
    R = float(Jt)
    e_inv = float(np.mean(inv))
    want = R * (1 - R) * (e_inv * (1 + 1 / (g - 1)) - 1 / (g - 1))
    got = ests.var(ddof=1)
    assert abs(got / want - 1) < 0.10, (got, want)
    # the empty-bin term is not negligible here: the 1/k form is off by > 15 %
    naive = R * (1 - R) * ((1 / k) * (1 + 1 / (g - 1)) - 1 / (g - 1))
    assert abs(naive / got - 1) > 0.15, (naive, got)


def test_oph_collision_probability_k1():
    """Eq. 5: with k = 1 bin the minima collide with
    probability J, within 3 standard errors over 4000 permutations."""
    rng = np.random.default_rng(21)
    V = 1 << 20
    A, B, Jt = _pair_with_union(400, 0.6, V, rng)
    offs, ids = make_csr([A, B])
    hits = 0
    n = 4000
    for seed in range(n):
        F = oracle.oph_sketch(offs, ids, V, 1, seed)
        hits += int(F[0, 0] == F[1, 0])
    p = float(Jt)
    assert abs(hits / n - p) < 3 * np.sqrt(p * (1 - p) / n)


def test_hoph_unbiased_joint_empty_dense():
    """Lemma 3: the HOPH estimator is unbiased; JointEmpty, sets dense
    relative to the bins (A.15), 3000 permutations, J = 0.5."""
    rng = np.random.default_rng(31)
    V, kp = 1 << 12, 16
    lay = oracle.hoph_layout(V, 1, 1, kp)
    L = len(lay)
    A, B, Jt = _pair_with_union(2048, 0.5, V, rng)
    offs, ids = make_csr([A, B])
    ests = []
    for seed in range(3000):
        H = oracle.hoph_sketch(offs, ids, V, lay, kp, seed)
        ests.append(oracle.hoph_estimate(H[0], H[1], L=L, kprime=kp, a=1, b=1, t_num=1, t_den=2,
                                         joint=True)["estimate"])
    ests = np.array(ests)
    se = ests.std(ddof=1) / np.sqrt(len(ests))
    assert abs(ests.mean() - float(Jt)) < 3 * se


def _hoph_r22_pair():
    """3 groups of k' = 4 (1:1: c = [2, 1, 1], D = 4); group 2 is empty on both
    sides, so it is excluded in either empty mode."""
    q = _sk([1, 2, 3, 4, None, None, None, None, 5, 6, 7, 8])
    s = _sk([1, 2, 3, 4, None, None, None, None, 5, 0, 7, None])
    return np.array(q, dtype=np.uint32), np.array(s, dtype=np.uint32)


@pytest.mark.parametrize("joint", [False, True])
def test_hoph_drop_renormalise_hand_example(joint):
    """R22 (S:416 'groups whose every bin is excluded are dropped and the
    remaining weights renormalized'): with group 2 fully excluded the
    estimate is (c1 m1/d1 + c3 m3/d3) / (c1 + c3), derived by hand:
      EitherEmpty: g1 m=4 of d=4, g3 m=2 of d=3 -> (2*1 + 1*2/3) / 3 = 8/9
      JointEmpty : g1 m=4 of d=4, g3 m=2 of d=4 -> (2*1 + 1*1/2) / 3 = 5/6
    (dividing by D = 4 instead would give 2/3 -- NotSimilar at T = 7/10 -- and
    5/8).  The filter path (compare_hoph, eps tiny) ends in the same record: the
    raw state S_2 = 8 keeps x = (T D k' - S_l) / W_l at 1.6 and 3.2, inside
    (0, k'], so only the last group decides; every group excluded -> UNDEFINED,
    NotSimilar."""
    q, s = _hoph_r22_pair()
    want = Fraction(5, 6) if joint else Fraction(8, 9)
    r = oracle.hoph_estimate(q, s, L=3, kprime=4, a=1, b=1, t_num=7, t_den=10, joint=joint)
    assert r["flags"] == 0
    assert r["estimate"] == pytest.approx(float(want), abs=1e-15)
    assert r["verdict"] == (want >= Fraction(7, 10))
    assert r["n_mb"] == 6
    assert r["n_excl"] == (4 if joint else 5)  # EitherEmpty 0 + 4 + 1; JointEmpty 0 + 4 + 0
    f = oracle.compare_hoph(q[None], s[None], L=3, kprime=4, a=1, b=1, t_num=7, t_den=10, eps=1e-300,
                            joint=joint)[0, 0]
    assert f["groups"] == 3 and f["flags"] == 0
    assert f["estimate"] == pytest.approx(float(want), abs=1e-15)
    assert f["verdict"] == r["verdict"]
    e = np.full(12, E, dtype=np.uint32)
    u = oracle.hoph_estimate(e, s, L=3, kprime=4, a=1, b=1, t_num=7, t_den=10, joint=False)
    assert u["flags"] & oracle.UNDEFINED and u["verdict"] == 0


def test_hoph_drop_renormalise_unbiased_sparse():
    """Lemma 3 with R22: JointEmpty, |V| = 2^16, k' = 16, L = 12 and a
    union of only 24 elements, so the deep groups hold no element of the
    union and are dropped in essentially every permutation.  Given the union's
    positions, every kept group's M_j / d_j is unbiased for J (which union
    elements are shared is exchangeable), so the renormalised mean is J within
    3 s.e. over 6000 permutations.  The same draws re-weighted with the
    dropped groups' weight left in the denominator (the "divide by D" misreading)
    miss J by more than 3 s.e., so this test would catch that mutant."""
    rng = np.random.default_rng(2222)
    V, kp = 1 << 16, 16
    lay = oracle.hoph_layout(V, 1, 1, kp)
    L = len(lay)
    assert L == 12
    c, D = oracle.hoph_weights(1, 1, L)
    A, B, Jt = _pair_with_union(24, 0.5, V, rng)
    offs, ids = make_csr([A, B])
    ests, mutant, dropped = [], [], 0
    for seed in range(6000):
        H = oracle.hoph_sketch(offs, ids, V, lay, kp, seed)
        ests.append(oracle.hoph_estimate(H[0], H[1], L=L, kprime=kp, a=1, b=1, t_num=1, t_den=2,
                                         joint=True)["estimate"])
        g0, g1 = H[0].reshape(L, kp), H[1].reshape(L, kp)
        both = (g0 == E) & (g1 == E)
        m = ((g0 == g1) & (g0 != E)).sum(1)
        d = kp - both.sum(1)
        keep = d > 0
        dropped += int((~keep).any())
        mutant.append(float(sum(c[j] * m[j] / d[j] for j in range(L) if keep[j]) / D))
    ests, mutant = np.array(ests), np.array(mutant)
    se = ests.std(ddof=1) / np.sqrt(len(ests))
    assert dropped >= 0.99 * len(ests)
    assert abs(ests.mean() - float(Jt)) < 3 * se
    assert abs(mutant.mean() - float(Jt)) > 3 * (mutant.std(ddof=1) / np.sqrt(len(mutant)))


# --------------------------------------------------------------------- Lemmas 1-3
def test_lemma1_lemma2_spec_examples():
    """r = 1/2, l = 2, N_mb = [1, 2] -> (1/4 + 2/8) 3 = 3/2; N_eb = [2, 0] ->
    (2/4) 3 = 3/2; all zeros -> 0."""
    from oracle import lemmas
    assert lemmas.hoph_aggregate([1, 2], Fraction(1, 2), 2) == Fraction(3, 2)
    assert lemmas.hoph_aggregate([2, 0], Fraction(1, 2), 2) == Fraction(3, 2)
    assert lemmas.hoph_aggregate([0, 0, 0], Fraction(1, 3), 3) == 0


def test_lemma1_equals_its_proof_first_line():
    """Lemma 1/2's closed form equals the proof's probability form times k_h = (l+1) k'
    (k_j = k'/r^j), exactly, on random counts for r in {1/2, 1/3, 2/3}: a wrong
    exponent (r^(2l) for r^(2l-1)) or factor ((l) for (l+1)) fails."""
    from oracle import lemmas
    rng = np.random.default_rng(91)
    for r in (Fraction(1, 2), Fraction(1, 3), Fraction(2, 3)):
        for l in (1, 2, 3, 5, 9):
            for _ in range(20):
                kp = int(rng.integers(1, 64))
                N = [int(x) for x in rng.integers(0, 2 * kp, size=l)]
                assert lemmas.hoph_aggregate(N, r, l) == \
                    lemmas.hoph_aggregate_probability(N, r, l, kp) * (l + 1) * kp


def test_lemma3_golden_and_terms():
    """Lemma 3 on the P:482 worked example, D1 vs D2 (groups [[1,1],[(x),0],[0,1]] vs
    [[1,2],[(x),0],[0,0]], k' = 2, r = 1/2): terms N_mb = [1, 1 + 1], N_eb = [0, 1 + 0] ->
    1/2 * 1/2 + 1/2 * 2/3 = 7/12 (S:467's 0.583 under R31); the last two groups' counts are
    summed."""
    from oracle import lemmas
    assert lemmas.lemma_terms([1, 1, 1]) == [1, 2]
    assert lemmas.lemma_terms([0, 1, 0]) == [0, 1]
    assert lemmas.hoph_lemma3_estimate([1, 2], [0, 1], Fraction(1, 2), 2, 2) == Fraction(7, 12)
    assert lemmas.hoph_lemma3_estimate([1, 2], [2, 0], Fraction(1, 2), 2, 2) is None


def test_lemma3_unbiased_joint_empty():
    """Lemma 3 ("the unbiased estimator"): under JointEmpty each term N_mb/(k - N_eb)
    is unbiased for J given the union's placement and the weights sum to 1 at r = 1/2, so
    over 3000 permutations the mean is J within 3 s.e. (1:1 HOPH over 2^12, k' = 16, a
    2048-element union: no term loses all its bins)."""
    from oracle import lemmas
    rng = np.random.default_rng(92)
    V, kp = 1 << 12, 16
    lay = oracle.hoph_layout(V, 1, 1, kp)
    L = len(lay)
    A, B, Jt = _pair_with_union(2048, 0.5, V, rng)
    offs, ids = make_csr([A, B])
    ests = []
    for seed in range(3000):
        H = oracle.hoph_sketch(offs, ids, V, lay, kp, seed)
        g0, g1 = H[0].reshape(L, kp), H[1].reshape(L, kp)
        m = ((g0 == g1) & (g0 != E)).sum(1).tolist()
        e = ((g0 == E) & (g1 == E)).sum(1).tolist()
        est = lemmas.hoph_lemma3_estimate(lemmas.lemma_terms(m), lemmas.lemma_terms(e), Fraction(1, 2), L - 1, kp)
        assert est is not None
        ests.append(float(est))
    ests = np.array(ests)
    se = ests.std(ddof=1) / np.sqrt(len(ests))
    assert abs(ests.mean() - float(Jt)) < 3 * se


# --------------------------------------------------------------------- MinWise
def test_minwise_properties():
    """S:283 full vocabulary -> all fingerprints 0; S:292 disjoint sets -> 0
    exactly; S:279 empty set flagged undefined; identical -> 1."""
    V = 64
    offs, ids = make_csr([range(V), range(0, 32), range(32, 64), []])
    F, fl = oracle.minwise_sketch(offs, ids, V, 50, 3)
    assert (F[0] == 0).all()
    assert list(fl) == [0, 0, 0, 1]
    r = oracle.compare_minwise(F, fl, F, fl, t_num=1, t_den=2)
    assert r[1, 2]["estimate"] == 0.0 and r[1, 2]["n_mb"] == 0
    assert r[1, 1]["estimate"] == 1.0 and r[1, 1]["verdict"] == 1
    assert r[3, 1]["flags"] & oracle.UNDEFINED and r[3, 3]["verdict"] == 0


def test_minwise_collision_rate():
    """Each MinWise position matches with probability J (Eq. 5 per
    permutation); k = 500 positions x 8 seeds, within 3 s.e. of J = 0.6."""
    rng = np.random.default_rng(41)
    V = 1 << 32
    A, B, Jt = _pair_with_union(300, 0.6, 1 << 24, rng)
    offs, ids = make_csr([A, B])
    eq = 0
    tot = 0
    for seed in range(8):
        F, _ = oracle.minwise_sketch(offs, ids, V, 500, seed)
        eq += int((F[0] == F[1]).sum())
        tot += 500
    p = float(Jt)
    assert abs(eq / tot - p) < 3 * np.sqrt(p * (1 - p) / tot)


# --------------------------------------------------------------------- Jaccard, invariants
def test_jaccard_brute_force():
    rng = np.random.default_rng(2)
    for _ in range(200):
        a = set(rng.integers(0, 50, size=int(rng.integers(0, 30))).tolist())
        b = set(rng.integers(0, 50, size=int(rng.integers(0, 30))).tolist())
        j, i, u = oracle.jaccard(sorted(a), sorted(b))
        assert (i, u) == (len(a & b), len(a | b))
        assert j == (len(a & b) / len(a | b) if (a | b) else None)


def test_pair_invariants_and_symmetry():
    """S:192 0 <= N_mb <= k - N_excl; JointEmpty excludes <= EitherEmpty;
    estimate in [0,1]; S:297/S:458 symmetry in the arguments."""
    from workloads import tiny
    w = tiny()
    p = w.params
    F = oracle.oph_sketch(w.offsets[:201], w.ids, w.vocab_size, p["k"], p["perm_seed"])
    re = oracle.compare_full(F, F, t_num=7, t_den=10, joint=False)
    rj = oracle.compare_full(F, F, t_num=7, t_den=10, joint=True)
    assert (re["n_excl"] >= rj["n_excl"]).all()
    for r in (re, rj):
        assert (r["n_mb"] <= p["k"] - r["n_excl"]).all()
        d = r["flags"] == 0
        assert ((r["estimate"][d] >= 0) & (r["estimate"][d] <= 1)).all()
        assert (r == r.T).all()


def test_goph_degeneracy_dense():
    """S:538 / S:618 on dense sets (R16, A.9): with eps = 1e-300 the filter can
    only stop on the certain guards, so GOPH verdicts equal full-OPH verdicts."""
    rng = np.random.default_rng(8)
    V, k, kp = 1 << 16, 256, 32
    sets = []
    base = rng.choice(V, size=4096, replace=False)
    for _ in range(40):
        J = rng.uniform(0.3, 1.0)
        keep = int(4096 * 2 * J / (1 + J))
        fresh = rng.choice(np.setdiff1d(np.arange(V), base), size=4096 - keep, replace=False)
        sets.append(np.concatenate([rng.choice(base, size=keep, replace=False), fresh]))
    offs, ids = make_csr(sets)
    F = oracle.oph_sketch(offs, ids, V, k, 1)
    assert (F != E).all()
    full = oracle.compare_full(F, F, t_num=7, t_den=10)
    go = oracle.compare_goph(F, F, n=k // kp, kprime=kp, t_num=7, t_den=10, eps=1e-300)
    assert (full["verdict"] == go["verdict"]).all()


def test_result_lists():
    """O12: threshold list sorted by (query, set_id); top-k by the
    exact estimate, ties to the smaller set_id (R27)."""
    recs = np.zeros((2, 5), dtype=oracle.REC_DTYPE)
    recs["verdict"][0] = [1, 0, 1, 1, 1]
    recs["n_mb"][0] = [3, 0, 4, 4, 2]
    recs["verdict"][1] = [0, 1, 0, 0, 0]
    recs["n_mb"][1] = [0, 5, 0, 0, 0]
    assert oracle.threshold_list(recs, 10) == [(0, 10), (0, 12), (0, 13), (0, 14), (1, 11)]
    assert oracle.topk_list(recs, 8, 2) == [(0, 2), (0, 3), (1, 1)]


# ----------------------------------------------------------------------------- shingling (ingestion, 8(f) rank 3)
def test_shingle_hash_known_answers():
    """FNV-1a 64 and splitmix64 against their published test vectors."""
    from oracle import shingle as sh
    assert sh.fnv1a64(b"") == 0xCBF29CE484222325
    assert sh.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert sh.fnv1a64(b"foobar") == 0x85944171F73967E8
    assert sh.splitmix64_stream(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_shingle_tokenizer_and_spec_examples():
    """Tokens == bytes.lower().split() (independent ASCII whitespace / case rules); SPEC examples."""
    import random
    from oracle import shingle as sh
    rng = random.Random(3)
    alphabet = b"abcXYZ \t\n\r\x0b\x0c01-'" + bytes([0xC3, 0xA9])
    for _ in range(300):
        text = bytes(rng.choice(alphabet) for _ in range(rng.randint(0, 60)))
        assert sh.tokens(text) == text.lower().split()
    V = 1 << 32
    assert len(sh.shingle_text(b"a b a b", 2, V, 7)) == 2            # "a b", "b a"
    assert sh.shingle_text(b"A\tB  a\nb", 2, V, 7) == sh.shingle_text(b"a b a b", 2, V, 7)
    assert sh.shingle_text(b"one two", 3, V, 7) == []                  # fewer than w tokens
    assert sh.shingle_text(b"", 1, V, 7) == []
    doc = b"the quick brown fox jumps over the lazy dog the quick brown fox"
    a = sh.shingle_text(doc, 3, V, 11)
    assert a == sh.shingle_text(doc, 3, V, 11) and a == sorted(set(a))
    assert len(sh.shingle_text(doc, 1, V, 11)) == len(set(doc.split()))  # w = 1: distinct tokens
    # the id is the seeded chain mod |V| (spot check of the definition, small |V|)
    toks = [b"x", b"y"]
    h = 5
    for t in toks:
        h = sh.mix64(h + sh.GOLDEN + sh.fnv1a64(t))
    assert sh.gram_id(toks, 1000, 5) == h % 1000
