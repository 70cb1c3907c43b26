"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports
every symbol include/ophgpu.h declares, validates arguments, builds the HOPH
layout like the oracle, and compiles the GOPH/HOPH rules into integer
thresholds that agree with the paper's rule evaluated exactly (Fractions) at
every reachable state."""
import ctypes
import os
import re
from fractions import Fraction

import numpy as np
import pytest

import oracle
import paper_1805_11254_b200 as og
from oracle import binomial

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    og.build()


def header_functions():
    src = open(os.path.join(ROOT, "include", "ophgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|oph_status|uint64_t)\s*(\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 12
    L = og.lib()
    for n in names:
        assert hasattr(L, n), n
    assert sorted(og.EXPORTS) == names


def test_status_strings_and_ld():
    assert og.status_string(og.OPH_OK) == "ok"
    assert "workspace" in og.status_string(og.OPH_ENOMEM)
    assert og.sketch_ld(1) == 32 and og.sketch_ld(32) == 32 and og.sketch_ld(33) == 64


def test_argument_validation_without_gpu():
    """Argument errors are reported before anything touches the device."""
    L = og.lib()
    assert L.oph_build_sketches(None, None, None, None, None, None, None, None, og.c_u64(0), None) == og.OPH_EINVAL
    sets = og.oph_sets(None, None, 0)
    perm = og.oph_perm(0, 1, 0, 0)  # vocab_size 0
    flat = og.oph_flat_layout(16, 4, 2)
    assert L.oph_build_sketches(ctypes.byref(sets), ctypes.byref(perm), ctypes.byref(flat), None, None, None, None, None,
                                og.c_u64(0), None) == og.OPH_EINVAL
    perm = og.oph_perm(16, 1, 0, 0)
    flat = og.oph_flat_layout(16, 32, 2)  # k > |V|
    dummy = og.c_vp(16)
    assert L.oph_build_sketches(ctypes.byref(sets), ctypes.byref(perm), ctypes.byref(flat), dummy, dummy, None, None,
                                None, og.c_u64(32), None) == og.OPH_EINVAL
    flat = og.oph_flat_layout(1 << 32, 1, 1)  # one bin of 2^32 ids leaves no room for the sentinels
    perm = og.oph_perm(1 << 32, 1, 0, 0)
    assert L.oph_build_sketches(ctypes.byref(sets), ctypes.byref(perm), ctypes.byref(flat), dummy, dummy, None, None,
                                None, og.c_u64(32), None) == og.OPH_EINVAL
    # compare: mismatched seeds are incompatible
    q = og.oph_sketches(dummy, dummy, None, 4, 32, 64, 0, 1, 1 << 16)
    s = og.oph_sketches(dummy, dummy, None, 4, 32, 64, 0, 2, 1 << 16)
    lay = og.oph_flat_layout(1 << 16, 64, 16)
    prm = og.params(7, 10, 1e-4)
    res = og.oph_results(dummy, 100, dummy, 0, 0)
    assert L.compare_full(ctypes.byref(q), ctypes.byref(s), og.c_u32(0), ctypes.byref(lay), ctypes.byref(prm),
                          ctypes.byref(res), dummy, ctypes.c_size_t(1 << 30), None) == og.OPH_EINCOMPAT
    bad = og.params(8, 7, 1e-4)  # T > 1
    s.seed = 1
    assert L.compare_full(ctypes.byref(q), ctypes.byref(s), og.c_u32(0), ctypes.byref(lay), ctypes.byref(bad),
                          ctypes.byref(res), dummy, ctypes.c_size_t(1 << 30), None) == og.OPH_EINVAL
    # a too-small workspace
    assert L.compare_full(ctypes.byref(q), ctypes.byref(s), og.c_u32(0), ctypes.byref(lay), ctypes.byref(prm),
                          ctypes.byref(res), dummy, ctypes.c_size_t(16), None) == og.OPH_ENOMEM
    with pytest.raises(og.OphError):
        og.oph_hier_layout_make(10, 1, 1, 8)  # |V| < 2k'


def test_hier_layout_matches_oracle():
    rng = np.random.default_rng(1)
    cases = [(17, 1, 1, 2), (1 << 16, 1, 1, 16), (1 << 32, 1, 1, 32), (1 << 20, 1, 2, 32), (1 << 20, 2, 1, 32)]
    cases += [(int(rng.integers(64, 10 ** 7)), int(rng.integers(1, 4)), int(rng.integers(1, 4)),
               int(rng.integers(1, 33))) for _ in range(100)]
    for V, a, b, kp in cases:
        try:
            want = oracle.hoph_layout(V, a, b, kp)
        except ValueError:
            with pytest.raises(og.OphError):
                og.oph_hier_layout_make(V, a, b, kp)
            continue
        got = og.oph_hier_layout_make(V, a, b, kp)
        assert got.groups() == want, (V, a, b, kp)


def _rule(x: Fraction, kp, T, lo, up):
    """The small-probability rule on x = M_ra (Alg. 1) or P_r k' (Alg. 2)."""
    if x <= 0:
        return 1
    if x > kp:
        return 2
    if x < kp * T:
        return 1 if lo[int(x)] else 0
    return 2 if up[-(-x.numerator // x.denominator)] else 0


def _compiled(acc, rej, st):
    return 1 if st >= acc else (2 if st <= rej else 0)


@pytest.mark.parametrize("kp,n,tn,td,eps", [(32, 8, 7, 10, 1e-4), (16, 4, 7, 10, 1e-4), (32, 16, 7, 10, 1e-4),
                                             (32, 8, 4, 5, 1e-4), (100, 10, 3, 5, 1e-4), (8, 12, 1, 2, 1e-2),
                                             (32, 16, 7, 10, 1e-3), (32, 16, 7, 10, 1e-5), (64, 4, 19, 20, 1e-4),
                                             (16, 6, 1, 1, 1e-4)])
def test_goph_thresholds_exhaustive(kp, n, tn, td, eps):
    """Every level, every M_c: compiled thresholds == Algorithm 1's rule (R10-R16)."""
    acc, rej, l0, w = og.plan_thresholds(og.OPH_METHOD_GOPH, n, kp, tn, td, eps)
    T = Fraction(tn, td)
    lo, up = binomial.small_probability_tables(kp, tn, td, eps)
    first = n
    for l in range(1, n):
        for Mc in range(0, l * kp + 1):
            want = _rule((n * kp * T - Mc) / (n - l), kp, T, lo, up)
            assert _compiled(acc[l - 1], rej[l - 1], Mc) == want, (l, Mc)
            if want and first == n:
                first = l
    assert l0 == first and w == [1] * n


def test_goph_thresholds_survey_values():
    """SURVEY A.3 (k'=32, n=8, T=0.7): levels 3..7 reject at <= 24, 55, 86, 117, 148; accept from 144, 156, 168."""
    acc, rej, l0, _ = og.plan_thresholds(og.OPH_METHOD_GOPH, 8, 32, 7, 10, 1e-4)
    assert rej == [-1, -1, 24, 55, 86, 117, 148] and acc[4:] == [144, 156, 168] and l0 == 3


@pytest.mark.parametrize("kp,L,a,b,tn,td,eps", [(32, 27, 1, 1, 7, 10, 1e-4), (16, 12, 1, 1, 7, 10, 1e-4),
                                                 (32, 15, 1, 1, 4, 5, 1e-4), (32, 10, 2, 1, 7, 10, 1e-4),
                                                 (16, 20, 1, 2, 7, 10, 1e-4), (100, 10, 1, 1, 3, 5, 1e-4)])
def test_hoph_thresholds_vs_mass_balance(kp, L, a, b, tn, td, eps):
    """Compiled HOPH thresholds == Algorithm 2's mass-balance rule (R19, R21)
    at every state near the boundaries, the low states and random states."""
    acc, rej, l0, c = og.plan_thresholds(og.OPH_METHOD_HOPH, L, kp, tn, td, eps, a, b)
    cw, D = oracle.hoph_weights(a, b, L)
    assert c == cw
    T = Fraction(tn, td)
    lo, up = binomial.small_probability_tables(kp, tn, td, eps)
    rng = np.random.default_rng(0)
    for l in range(1, L):
        W = D - sum(c[:l])
        smax = kp * sum(c[:l])
        states = set(range(0, min(smax, 300) + 1)) | {smax}
        for t in (acc[l - 1], rej[l - 1]):
            if 0 <= t <= smax:
                states |= {max(0, t - 2), max(0, t - 1), t, min(smax, t + 1), min(smax, t + 2)}
        states |= set(int(x) for x in rng.integers(0, smax + 1, size=200))
        for S in states:
            x = (T * D * kp - S) / W
            assert _compiled(acc[l - 1], rej[l - 1], S) == _rule(x, kp, T, lo, up), (l, S)
    assert l0 == 1


def test_hoph_thresholds_survey_values():
    """SURVEY A.7 (1:1, k'=32, T=0.7): level 1 rejects S/c1 <= 13.8 (M_1 <= 13); level 2 (38.8, 29.3)."""
    acc, rej, _, c = og.plan_thresholds(og.OPH_METHOD_HOPH, 27, 32, 7, 10, 1e-4)
    c1 = c[0]
    assert rej[0] // c1 == 13 and acc[0] == 2 ** 64 - 1
    assert Fraction(rej[1], c1) < Fraction(293, 10) <= Fraction(rej[1] + 1, c1)
    assert Fraction(acc[1] - 1, c1) < Fraction(388, 10) <= Fraction(acc[1], c1)


def test_workspace_size_monotone():
    a = og.oph_workspace_size(og.OPH_METHOD_HOPH, 1000, 200_000, 864, 0)
    b = og.oph_workspace_size(og.OPH_METHOD_HOPH, 1000, 200_000, 864, 10 ** 8)
    c = og.oph_workspace_size(og.OPH_METHOD_FULL, 1000, 200_000, 256, 0)
    assert b > a > c > 0
