"""The multi-GPU path on one GPU (SURVEY 4 "fake multi-GPU on one GPU", 8(e)):
the collection is split into 8 contiguous shards, each shard is sketched and
scored on its own with set IDs offset by its shard base (what rank r does),
the per-shard hit records are concatenated (the gather) and merged by
topk_or_threshold_results (rank 0).  The merged hit lists must be byte-
identical to the unsharded run's and equal to the oracle's."""
import numpy as np
import pytest

import oracle
import paper_1805_11254_b200 as og
from paper_1805_11254_b200 import dist as odist
from workloads import text_like, tiny

from gpu_helpers import oracle_records, subview

pytestmark = pytest.mark.gpu

SHARDS = 8


@pytest.fixture(scope="module", autouse=True)
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    og.build()


def _surv(q, shard):
    return min(((q.n_sets + 31) // 32) * 32 * shard.n_sets, 1 << 26)


def _score(method, w, q, shard, base, prm, flat, hier, cap):
    """One shard's compare call: sketches of the shard, threshold records appended."""
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    sets = og.SetCollection.from_numpy(shard.offsets, shard.ids)
    res = og.Results(cap)
    if method == "minwise":
        s = og.minwise_build_sketches(sets, V, seed, p["mw_k"])
        og.compare_minwise(q, s, prm, res, set_id_base=base)
    else:
        so, sh = og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier)
        if method == "full":
            og.compare_full(q, so, flat, prm, res, set_id_base=base)
        elif method == "goph":
            og.compare_goph(q, so, flat, prm, res, set_id_base=base, survivor_capacity=_surv(q, shard))
        else:
            og.compare_hoph(q, sh, hier, prm, res, set_id_base=base, survivor_capacity=_surv(q, shard))
    n = res.n()
    assert n <= cap
    return res.hits[: n * og.HIT_DTYPE.itemsize].clone(), n


def _merge(chunks):
    import torch
    allh = torch.cat([c for c, _ in chunks]) if chunks else None
    n = sum(m for _, m in chunks)
    src = og.Results(max(n, 1))
    if n:
        src.hits[: allh.numel()].copy_(allh)
    out = og.Results(max(n, 1))
    og.topk_or_threshold_results(src, n, og.OPH_SELECT_THRESHOLD, out)
    assert out.n() == n
    return out.numpy(n)


def _run(w, methods, n_query_sample, strategy):
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    flat = og.flat_layout(V, p["k"], p["kprime"])
    hier = og.oph_hier_layout_make(V, p["a"], p["b"], p["hoph_kprime"])
    prm = og.params(p["t_num"], p["t_den"], p["eps"], strategy=strategy)
    qsets = og.SetCollection.from_numpy(w.q_offsets, w.q_ids)
    qo, qh = og.oph_build_sketches(qsets, V, seed, flat=flat, hier=hier)
    qmw = og.minwise_build_sketches(qsets, V, seed, p["mw_k"])
    glay = oracle.hoph_layout(V, p["a"], p["b"], p["hoph_kprime"])
    nq = n_query_sample
    QF = oracle.oph_sketch(w.q_offsets[: nq + 1], w.q_ids, V, p["k"], seed)
    QH = oracle.hoph_sketch(w.q_offsets[: nq + 1], w.q_ids, V, glay, p["hoph_kprime"], seed)
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    cap = 1 << 22
    for m in methods:
        q = {"full": qo, "goph": qo, "hoph": qh, "minwise": qmw}[m]
        whole = _merge([_score(m, w, q, w, 0, prm, flat, hier, cap)])
        chunks = []
        for r in range(SHARDS):
            lo, hi = odist.shard_range(w.n_sets, r, SHARDS)
            chunks.append(_score(m, w, q, w.slice_sets(lo, hi), lo, prm, flat, hier, cap))
        merged = _merge(chunks[::-1])  # the gather order does not matter
        assert merged.tobytes() == whole.tobytes(), m
        assert len(whole) > 0, m
        # the oracle on the first nq queries over every set
        if m == "minwise":
            MW, fl = oracle.minwise_sketch(w.offsets, w.ids, V, p["mw_k"], seed)
            QMW, qfl = oracle.minwise_sketch(w.q_offsets[: nq + 1], w.q_ids, V, p["mw_k"], seed)
            want = oracle_records(m, QMW, MW, qflags=qfl, sflags=fl, t_num=p["t_num"], t_den=p["t_den"])
        elif m == "hoph":
            H = oracle.hoph_sketch(w.offsets, w.ids, V, glay, p["hoph_kprime"], seed)
            want = oracle_records(m, QH, H, kprime=p["hoph_kprime"], L=len(glay), **kw)
        else:
            F = oracle.oph_sketch(w.offsets, w.ids, V, p["k"], seed)
            want = oracle_records(m, QF, F, k=p["k"], kprime=p["kprime"], **kw)
        sel = merged[merged["query"] < nq]
        assert [(int(a), int(b)) for a, b in zip(sel["query"], sel["set_id"])] == oracle.threshold_list(want), m
        rec = want[sel["query"].astype(np.int64), sel["set_id"].astype(np.int64)]
        for f in ("n_mb", "n_excl", "groups", "verdict", "flags"):
            assert (sel[f].astype(np.int64) == rec[f].astype(np.int64)).all(), (m, f)


@pytest.mark.parametrize("strategy", [og.OPH_STRATEGY_BRUTE, og.OPH_STRATEGY_PROBE])
def test_tiny_sharded_equals_unsharded(strategy):
    w = tiny()
    _run(w, ["full", "goph", "hoph", "minwise"], w.n_queries, strategy)


def test_text_like_sharded_equals_unsharded():
    """text-like (configs[1]) in 8 shards of 25,000 sets, all 1,000 queries; the oracle
    checks the first 16 queries against every set."""
    w = text_like()
    _run(w, ["full", "goph", "hoph", "minwise"], 16, og.OPH_STRATEGY_AUTO)
