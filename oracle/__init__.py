"""CPU oracle for OPH / GOPH / HOPH / MinWise near-duplicate scoring.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import this package.
The product package `paper_1805_11254_b200` never imports it and shares no
code with it.

The arithmetic lives in plain C (`oracle.c`, exact integers / rationals,
one function per step of the paper, each citing its passage) and in
`binomial.py` (exact rational binomial tails).  This module only marshals
numpy arrays.  Sketch arrays are set-major here: [n_sets][n_bins] uint32,
EMPTY = 0xFFFFFFFF.

Parity pins: tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import binomial  # noqa: F401
from .binomial import lower_tail, small_probability_tables, upper_tail  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

EMPTY = 0xFFFFFFFF
UNDEFINED = 1
EARLY = 2

REC_DTYPE = np.dtype([("n_mb", "<u4"), ("n_excl", "<u4"), ("groups", "<u4"), ("verdict", "<u4"),
                      ("flags", "<u4"), ("pad", "<u4"), ("estimate", "<f8")])


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, OpenMP, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fopenmp", "-ffp-contract=off",
                               "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.orc_jaccard.restype = ctypes.c_double
        _lib.orc_hoph_layout.restype = ctypes.c_uint32
        _lib.orc_num_threads.restype = ctypes.c_int
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _u64(x):
    return ctypes.c_uint64(int(x))


def _u32(x):
    return ctypes.c_uint32(int(x))


def num_threads() -> int:
    return int(lib().orc_num_threads())


def _csr(offsets, ids):
    return np.ascontiguousarray(offsets, dtype=np.uint64), np.ascontiguousarray(ids, dtype=np.uint32)


# ---------------------------------------------------------------- O1 psi
def psi(x, vocab_size: int, seed: int, identity: bool = False) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.uint64)
    out = np.empty_like(x)
    lib().orc_psi_apply(_u64(vocab_size), _u64(seed), ctypes.c_int(int(identity)), _p(x), _u64(len(x)), _p(out))
    return out


# ---------------------------------------------------------------- O3 / O5 / O6 sketches
def oph_sketch(offsets, ids, vocab_size: int, k: int, seed: int, identity: bool = False) -> np.ndarray:
    offsets, ids = _csr(offsets, ids)
    n = len(offsets) - 1
    out = np.empty((n, k), dtype=np.uint32)
    lib().orc_oph_sketch(_p(offsets), _p(ids), _u64(n), _u64(vocab_size), _u32(k), _u64(seed),
                         ctypes.c_int(int(identity)), _p(out))
    return out


def hoph_layout(vocab_size: int, a: int, b: int, kprime: int) -> list[tuple[int, int]]:
    start = np.zeros(64, dtype=np.uint64)
    length = np.zeros(64, dtype=np.uint64)
    L = lib().orc_hoph_layout(_u64(vocab_size), _u32(a), _u32(b), _u32(kprime), _u32(64), _p(start), _p(length))
    if L == 0:
        raise ValueError("hoph_layout: invalid arguments or more than 64 groups")
    return [(int(start[i]), int(length[i])) for i in range(L)]


def hoph_sketch(offsets, ids, vocab_size: int, layout, kprime: int, seed: int, identity: bool = False) -> np.ndarray:
    offsets, ids = _csr(offsets, ids)
    n = len(offsets) - 1
    L = len(layout)
    gs = np.array([g[0] for g in layout], dtype=np.uint64)
    gl = np.array([g[1] for g in layout], dtype=np.uint64)
    out = np.empty((n, L * kprime), dtype=np.uint32)
    lib().orc_hoph_sketch(_p(offsets), _p(ids), _u64(n), _u64(vocab_size), _u32(L), _p(gs), _p(gl),
                          _u32(kprime), _u64(seed), ctypes.c_int(int(identity)), _p(out))
    return out


def minwise_sketch(offsets, ids, vocab_size: int, k: int, seed: int):
    offsets, ids = _csr(offsets, ids)
    n = len(offsets) - 1
    out = np.empty((n, k), dtype=np.uint32)
    flags = np.empty(n, dtype=np.uint8)
    lib().orc_minwise_sketch(_p(offsets), _p(ids), _u64(n), _u64(vocab_size), _u32(k), _u64(seed),
                             _p(out), _p(flags))
    return out, flags


def hoph_weights(a: int, b: int, L: int):
    """Integer nominal weights c_j (j = 1..L) over D = (a+b)^(L-1)."""
    c = np.zeros(L, dtype=np.int64)
    D = np.zeros(1, dtype=np.int64)
    lib().orc_hoph_weights(_u32(a), _u32(b), _u32(L), _p(c), _p(D))
    return [int(x) for x in c], int(D[0])


# ---------------------------------------------------------------- O11 Jaccard
def jaccard(a, b):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    i = ctypes.c_uint64()
    u = ctypes.c_uint64()
    j = lib().orc_jaccard(_p(a), _u64(len(a)), _p(b), _u64(len(b)), ctypes.byref(i), ctypes.byref(u))
    return (None if j < 0 else j), int(i.value), int(u.value)


# ---------------------------------------------------------------- O7 / O9 / O10 / MinWise
def _recs(nq, ns):
    return np.zeros((nq, ns), dtype=REC_DTYPE)


def compare_full(Q, S, *, t_num, t_den, joint=False, groups=0):
    Q = np.ascontiguousarray(Q, dtype=np.uint32)
    S = np.ascontiguousarray(S, dtype=np.uint32)
    k = Q.shape[1]
    assert S.shape[1] == k
    out = _recs(Q.shape[0], S.shape[0])
    lib().orc_compare_full(_p(Q), _u64(Q.shape[0]), _p(S), _u64(S.shape[0]), _u32(k), _u32(groups),
                           ctypes.c_int(int(joint)), _u32(t_num), _u32(t_den), _p(out))
    return out


def compare_goph(Q, S, *, n, kprime, t_num, t_den, eps, joint=False, trace=False, empty_aware=False):
    """Algorithm 1 (O9); empty_aware: the empty-aware variant (O9e, E1-E4)."""
    Q = np.ascontiguousarray(Q, dtype=np.uint32)
    S = np.ascontiguousarray(S, dtype=np.uint32)
    assert Q.shape[1] == S.shape[1] == n * kprime
    lo, up = small_probability_tables(kprime, t_num, t_den, eps)
    lo = np.frombuffer(lo, dtype=np.uint8).copy()
    up = np.frombuffer(up, dtype=np.uint8).copy()
    out = _recs(Q.shape[0], S.shape[0])
    tr = np.zeros((Q.shape[0], S.shape[0], n, 2), dtype=np.int64) if trace else None
    lib().orc_compare_goph(_p(Q), _u64(Q.shape[0]), _p(S), _u64(S.shape[0]), _u32(n), _u32(kprime),
                           ctypes.c_int(int(joint)), _u32(t_num), _u32(t_den), _p(lo), _p(up), _p(out), _p(tr),
                           ctypes.c_int(int(empty_aware)))
    return (out, tr) if trace else out


def compare_hoph(Q, S, *, L, kprime, a, b, t_num, t_den, eps, joint=False, trace=False, empty_aware=False):
    Q = np.ascontiguousarray(Q, dtype=np.uint32)
    S = np.ascontiguousarray(S, dtype=np.uint32)
    assert Q.shape[1] == S.shape[1] == L * kprime and L <= 64
    lo, up = small_probability_tables(kprime, t_num, t_den, eps)
    lo = np.frombuffer(lo, dtype=np.uint8).copy()
    up = np.frombuffer(up, dtype=np.uint8).copy()
    out = _recs(Q.shape[0], S.shape[0])
    tr = np.zeros((Q.shape[0], S.shape[0], L, 2), dtype=np.int64) if trace else None
    lib().orc_compare_hoph(_p(Q), _u64(Q.shape[0]), _p(S), _u64(S.shape[0]), _u32(L), _u32(kprime),
                           _u32(a), _u32(b), ctypes.c_int(int(joint)), _u32(t_num), _u32(t_den),
                           _p(lo), _p(up), _p(out), _p(tr), ctypes.c_int(int(empty_aware)))
    return (out, tr) if trace else out


def hoph_estimate(q, s, *, L, kprime, a, b, t_num, t_den, joint=False):
    """The HOPH estimator of one sketch pair (all groups, no filter)."""
    q = np.ascontiguousarray(q, dtype=np.uint32)
    s = np.ascontiguousarray(s, dtype=np.uint32)
    out = np.zeros(1, dtype=REC_DTYPE)
    lib().orc_hoph_estimate(_p(q), _p(s), _u32(L), _u32(kprime), _u32(a), _u32(b), ctypes.c_int(int(joint)),
                            _u32(t_num), _u32(t_den), _p(out))
    return out[0]


def compare_minwise(Q, qflags, S, sflags, *, t_num, t_den):
    Q = np.ascontiguousarray(Q, dtype=np.uint32)
    S = np.ascontiguousarray(S, dtype=np.uint32)
    qf = np.ascontiguousarray(qflags, dtype=np.uint8)
    sf = np.ascontiguousarray(sflags, dtype=np.uint8)
    k = Q.shape[1]
    out = _recs(Q.shape[0], S.shape[0])
    lib().orc_compare_minwise(_p(Q), _p(qf), _u64(Q.shape[0]), _p(S), _p(sf), _u64(S.shape[0]), _u32(k),
                              _u32(t_num), _u32(t_den), _p(out))
    return out


# ---------------------------------------------------------------- O12 result lists
def threshold_list(recs, set_id_base: int = 0):
    """Similar pairs as (query, set_id), sorted by (query, set_id)."""
    q, s = np.nonzero(recs["verdict"] == 1)
    order = np.lexsort((s, q))
    return [(int(q[i]), int(s[i]) + set_id_base) for i in order]


def topk_list(recs, k_bins: int, topk: int, set_id_base: int = 0):
    """Per query: the Similar pairs with a defined estimate, ordered by the
    exact rational estimate n_mb / (k_bins - n_excl) descending, ties by the
    smaller set_id; the first `topk` of each query (R27).  For
    full-OPH or MinWise records (MinWise: n_excl = 0).  Returns (query, set_id)
    pairs in output order."""
    from fractions import Fraction
    out = []
    for q in range(recs.shape[0]):
        cand = []
        for s in np.nonzero(recs["verdict"][q] == 1)[0]:
            r = recs[q, s]
            if int(r["flags"]) & UNDEFINED:
                continue
            cand.append((-Fraction(int(r["n_mb"]), k_bins - int(r["n_excl"])), int(s)))
        cand.sort()
        out.extend((q, s + set_id_base) for _, s in cand[:topk])
    return out
