"""Shared helpers of the -m gpu parity tests: run the CUDA path (through the
C-ABI binding) and the oracle on the same seeded inputs, compare records."""
from __future__ import annotations

import numpy as np

import oracle
import paper_1805_11254_b200 as og

REC_FIELDS = ("n_mb", "n_excl", "groups", "verdict", "flags")
EST_TOL = 1e-6  # B.north_star: floating-point estimates within 1e-6 absolute


def gpu_build(offsets, ids, V, seed, k=None, kprime=None, hier=None, identity=False):
    sets = og.SetCollection.from_numpy(offsets, ids)
    flat = og.flat_layout(V, k, kprime) if k else None
    so, sh = og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier, identity=identity)
    return sets, so, sh


def gpu_dense(method, q, s, *, layout=None, t_num, t_den, eps=1e-4, joint=False, survivor_capacity=0,
              strategy=og.OPH_STRATEGY_AUTO):
    """Dense per-pair records [n_q, n_s] from the GPU (AUTO: the BITMAP join where it
    applies -- |V| <= 2^23, not MinWise -- else the BRUTE scan)."""
    res = og.Results(q.n_sets * s.n_sets, dense=True)
    prm = og.params(t_num, t_den, eps, joint, strategy,
                    variant=og.OPH_VARIANT_EMPTY_AWARE if method in ("goph_e", "hoph_e") else 0)
    if method == "full":
        og.compare_full(q, s, layout, prm, res)
    elif method in ("goph", "goph_e"):
        og.compare_goph(q, s, layout, prm, res, survivor_capacity=survivor_capacity)
    elif method in ("hoph", "hoph_e"):
        og.compare_hoph(q, s, layout, prm, res, survivor_capacity=survivor_capacity)
    elif method == "minwise":
        og.compare_minwise(q, s, prm, res)
    return res.numpy().reshape(q.n_sets, s.n_sets)


def assert_records_equal(gpu, orc, what=""):
    """Bit-exact integer fields, estimates within EST_TOL where defined."""
    assert gpu.shape == orc.shape, what
    for f in REC_FIELDS:
        bad = np.nonzero(gpu[f].astype(np.int64) != orc[f].astype(np.int64))
        if len(bad[0]):
            i, j = bad[0][0], bad[1][0]
            raise AssertionError(f"{what}: field {f} differs at {len(bad[0])} pairs; first ({i},{j}): "
                                 f"gpu {gpu[i, j]} oracle {orc[i, j]}")
    has = (orc["flags"] == 0)
    if has.any():
        err = np.abs(gpu["estimate"][has].astype(np.float64) - orc["estimate"][has])
        assert err.max() <= EST_TOL, f"{what}: estimate error {err.max()}"
    assert (gpu["estimate"][~has] == -1.0).all(), what
    q, s = np.nonzero(np.ones(gpu.shape, dtype=bool))
    assert (gpu["query"].ravel() == q).all() and (gpu["set_id"].ravel() == s).all(), what


def gpu_threshold_hits(method, q, s, *, layout=None, t_num, t_den, eps=1e-4, joint=False, capacity=1 << 20,
                       set_id_base=0, survivor_capacity=0, strategy=og.OPH_STRATEGY_AUTO):
    """Sorted threshold hit list from the GPU (compare + topk_or_threshold_results)."""
    res = og.Results(capacity)
    prm = og.params(t_num, t_den, eps, joint, strategy,
                    variant=og.OPH_VARIANT_EMPTY_AWARE if method in ("goph_e", "hoph_e") else 0)
    if method == "full":
        og.compare_full(q, s, layout, prm, res, set_id_base=set_id_base)
    elif method in ("goph", "goph_e"):
        og.compare_goph(q, s, layout, prm, res, set_id_base=set_id_base, survivor_capacity=survivor_capacity)
    elif method in ("hoph", "hoph_e"):
        og.compare_hoph(q, s, layout, prm, res, set_id_base=set_id_base, survivor_capacity=survivor_capacity)
    elif method == "minwise":
        og.compare_minwise(q, s, prm, res, set_id_base=set_id_base)
    n = res.n()
    assert n <= capacity
    out = og.Results(max(n, 1))
    og.topk_or_threshold_results(res, n, og.OPH_SELECT_THRESHOLD, out)
    m = out.n()
    assert m == n
    return out.numpy(m)


def oracle_records(method, Q, S, *, t_num, t_den, eps=1e-4, joint=False, k=None, kprime=None, L=None, a=1, b=1,
                   qflags=None, sflags=None, strategy=None):
    """The oracle's dense records (`strategy` is the GPU's and ignored here)."""
    if method == "full":
        return oracle.compare_full(Q, S, t_num=t_num, t_den=t_den, joint=joint, groups=k // kprime)
    if method in ("goph", "goph_e"):
        return oracle.compare_goph(Q, S, n=k // kprime, kprime=kprime, t_num=t_num, t_den=t_den, eps=eps, joint=joint,
                                   empty_aware=method == "goph_e")
    if method in ("hoph", "hoph_e"):
        return oracle.compare_hoph(Q, S, L=L, kprime=kprime, a=a, b=b, t_num=t_num, t_den=t_den, eps=eps, joint=joint,
                                   empty_aware=method == "hoph_e")
    if method == "minwise":
        return oracle.compare_minwise(Q, qflags, S, sflags, t_num=t_num, t_den=t_den)
    raise ValueError(method)


def masks_from_values(vals: np.ndarray) -> np.ndarray:
    """Expected empty masks [n, ceil(nb/32)] of set-major sketches (bit b%32 of word b/32)."""
    n, nb = vals.shape
    nw = (nb + 31) // 32
    out = np.zeros((n, nw), dtype=np.uint64)
    for b in range(nb):
        out[:, b // 32] |= (vals[:, b] == oracle.EMPTY).astype(np.uint64) << np.uint64(b % 32)
    return out.astype(np.uint32)


def subview(sk: og.Sketches, n: int) -> og.Sketches:
    """The first n columns of a sketch matrix as its own view."""
    import dataclasses
    return dataclasses.replace(sk, n_sets=n)
