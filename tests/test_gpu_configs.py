"""Parity at BASELINE.json's full sizes for configs[2] (image-like), configs[3]
(one per-GPU shard of scale) and configs[4] (similarity sweep), in the launch
configuration bench.py uses: all queries x all sets in threshold mode; the
oracle checks the hit lists of sampled queries against every set, dense
records of a contiguous query block, and the sketches of every set.  MinWise
(k = 512 permutations: 4x10^11 oracle evaluations per 10^6 sets) is checked on
a sampled 4,000-set sub-collection."""
import numpy as np
import pytest

import oracle
import paper_1805_11254_b200 as og

from gpu_helpers import assert_records_equal, gpu_dense, gpu_threshold_hits, masks_from_values, oracle_records, subview

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module", autouse=True)
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    og.build()


def _check_sketches_chunked(gpu_sk, orc, chunk=100_000):
    vals = gpu_sk.values
    emp = gpu_sk.empty
    for c0 in range(0, gpu_sk.n_sets, chunk):
        c1 = min(gpu_sk.n_sets, c0 + chunk)
        g = vals[:, c0:c1].cpu().numpy().view(np.uint32).T
        assert (g == orc[c0:c1]).all(), f"sketch mismatch in sets [{c0},{c1})"
        ge = emp[:, c0:c1].cpu().numpy().view(np.uint32).T
        assert (ge == masks_from_values(orc[c0:c1])).all(), f"mask mismatch in sets [{c0},{c1})"


def check_config(w, sample, strategy, methods=("full", "goph", "hoph"), dense_q=4, hit_queries=None):
    """hit_queries: score only the first hit_queries queries in threshold mode
    (the sweep's all-similar collections give ~10^8-10^9 hits for all queries)."""
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    hier = og.oph_hier_layout_make(V, p["a"], p["b"], p["hoph_kprime"])
    flat = og.flat_layout(V, p["k"], p["kprime"])
    sets = og.SetCollection.from_numpy(w.offsets, w.ids)
    qs = og.SetCollection.from_numpy(w.q_offsets, w.q_ids)
    so, sh = og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier)
    qo, qh = og.oph_build_sketches(qs, V, seed, flat=flat, hier=hier)
    glay = oracle.hoph_layout(V, p["a"], p["b"], p["hoph_kprime"])
    F = oracle.oph_sketch(w.offsets, w.ids, V, p["k"], seed)
    _check_sketches_chunked(so, F)
    H = oracle.hoph_sketch(w.offsets, w.ids, V, glay, p["hoph_kprime"], seed)
    _check_sketches_chunked(sh, H)
    QF = oracle.oph_sketch(w.q_offsets, w.q_ids, V, p["k"], seed)
    QH = oracle.hoph_sketch(w.q_offsets, w.q_ids, V, glay, p["hoph_kprime"], seed)
    assert (qo.numpy() == QF).all() and (qh.numpy() == QH).all()
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    if hit_queries is not None:
        qo_t, qh_t = subview(qo, hit_queries), subview(qh, hit_queries)
        assert max(sample) < hit_queries
    else:
        qo_t, qh_t = qo, qh
    for m in methods:
        if m == "hoph":
            hits = gpu_threshold_hits(m, qh_t, sh, layout=hier, strategy=strategy, capacity=1 << 26, **kw)
            want = oracle_records(m, QH[sample], H, kprime=p["hoph_kprime"], L=len(glay), **kw)
            dense = gpu_dense(m, subview(qh, dense_q), sh, layout=hier, **kw)
            dwant = oracle_records(m, QH[:dense_q], H, kprime=p["hoph_kprime"], L=len(glay), **kw)
        else:
            hits = gpu_threshold_hits(m, qo_t, so, layout=flat, strategy=strategy, capacity=1 << 26, **kw)
            want = oracle_records(m, QF[sample], F, k=p["k"], kprime=p["kprime"], **kw)
            dense = gpu_dense(m, subview(qo, dense_q), so, layout=flat, **kw)
            dwant = oracle_records(m, QF[:dense_q], F, k=p["k"], kprime=p["kprime"], **kw)
        sset = set(sample)
        got = [(int(h["query"]), int(h["set_id"])) for h in hits if int(h["query"]) in sset]
        assert got == [(sample[q], s) for q, s in oracle.threshold_list(want)], m
        assert_records_equal(dense, dwant, f"{w.name} {m}")
    # MinWise on a sampled sub-collection
    rng = np.random.default_rng(0)
    sub = np.sort(rng.choice(w.n_sets, size=min(4000, w.n_sets), replace=False))
    sub_sets = [w.set_ids(int(s)) for s in sub]
    soff = np.zeros(len(sub) + 1, dtype=np.uint64)
    np.cumsum([len(x) for x in sub_sets], out=soff[1:])
    sids = np.concatenate(sub_sets)
    nq = 64
    qoff = w.q_offsets[: nq + 1]
    mw = og.minwise_build_sketches(og.SetCollection.from_numpy(soff, sids), V, seed, p["mw_k"])
    qmw = og.minwise_build_sketches(og.SetCollection.from_numpy(qoff, w.q_ids[: int(qoff[-1])]), V, seed, p["mw_k"])
    MW, fl = oracle.minwise_sketch(soff, sids, V, p["mw_k"], seed)
    QMW, qfl = oracle.minwise_sketch(qoff, w.q_ids, V, p["mw_k"], seed)
    assert (mw.numpy() == MW).all() and (qmw.numpy() == QMW).all()
    assert_records_equal(gpu_dense("minwise", qmw, mw, t_num=p["t_num"], t_den=p["t_den"]),
                         oracle_records("minwise", QMW, MW, qflags=qfl, sflags=fl, t_num=p["t_num"], t_den=p["t_den"]),
                         f"{w.name} minwise")


def test_image_like_full_size():
    from workloads.gen_gpu import image_like
    w = image_like()
    assert w.n_sets == 1_000_000 and w.n_queries == 4096
    # the bench's strategy (BITMAP, blocks of 2,048 queries for full OPH / GOPH); samples on
    # both sides of every block boundary
    check_config(w, sample=[0, 1, 2, 1000, 2047, 2048, 3071, 4095], strategy=og.OPH_STRATEGY_BITMAP)


def test_scale_shard_full_size():
    from workloads.gen_gpu import scale_shard
    w = scale_shard(shard=0)
    assert w.n_sets == 1_250_000 and w.n_queries == 16384
    check_config(w, sample=[0, 5, 777, 8191, 16383], strategy=og.OPH_STRATEGY_AUTO)


@pytest.mark.parametrize("method", ["goph", "hoph"])
def test_probe_survivor_overflow_redo(method):
    """PROBE first scores every query at once; on a high-similarity collection
    the survivor list overflows a minimal workspace, the hit counter is rolled
    back and the queries are redone in worst-case-sized chunks: the hit list
    still equals the oracle's exactly."""
    from workloads.gen_gpu import sweep
    w = sweep(0.9, n_sets=20_000, n_queries=128)
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    hier = og.oph_hier_layout_make(V, 1, 1, p["hoph_kprime"])
    flat = og.flat_layout(V, p["k"], p["kprime"])
    so, sh = og.oph_build_sketches(og.SetCollection.from_numpy(w.offsets, w.ids), V, seed, flat=flat, hier=hier)
    qo, qh = og.oph_build_sketches(og.SetCollection.from_numpy(w.q_offsets, w.q_ids), V, seed, flat=flat, hier=hier)
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    cap = 32 * w.n_sets
    if method == "hoph":
        glay = oracle.hoph_layout(V, 1, 1, p["hoph_kprime"])
        H = oracle.hoph_sketch(w.offsets, w.ids, V, glay, p["hoph_kprime"], seed)
        QH = oracle.hoph_sketch(w.q_offsets, w.q_ids, V, glay, p["hoph_kprime"], seed)
        want = oracle_records(method, QH, H, kprime=p["hoph_kprime"], L=len(glay), **kw)
        hits = gpu_threshold_hits(method, qh, sh, layout=hier, strategy=og.OPH_STRATEGY_PROBE, capacity=1 << 23,
                                  survivor_capacity=cap, **kw)
    else:
        F = oracle.oph_sketch(w.offsets, w.ids, V, p["k"], seed)
        QF = oracle.oph_sketch(w.q_offsets, w.q_ids, V, p["k"], seed)
        want = oracle_records(method, QF, F, k=p["k"], kprime=p["kprime"], **kw)
        hits = gpu_threshold_hits(method, qo, so, layout=flat, strategy=og.OPH_STRATEGY_PROBE, capacity=1 << 23,
                                  survivor_capacity=cap, **kw)
    assert [(int(h["query"]), int(h["set_id"])) for h in hits] == oracle.threshold_list(want)


@pytest.mark.parametrize("jmax", [0.9, 0.5, 0.2])
def test_sweep(jmax):
    """configs[4] at its full size (2 x 10^6 sets per Jmax), the bench's BITMAP strategy."""
    from workloads.gen_gpu import sweep
    w = sweep(jmax, n_sets=2_000_000)
    check_config(w, sample=[0, 3, 17, 31], strategy=og.OPH_STRATEGY_BITMAP, dense_q=2, hit_queries=32)


@pytest.mark.parametrize("shard", [1, 2, 3, 4, 5, 6, 7])
def test_scale_other_shards(shard):
    """configs[3]'s other seven per-GPU shards: every sketch == the oracle's, and the hit lists
    of two sampled queries over all 1.25 x 10^6 sets (AUTO: the PROBE join) == the oracle's."""
    from workloads.gen_gpu import scale_shard
    w = scale_shard(shard=shard)
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    hier = og.oph_hier_layout_make(V, p["a"], p["b"], p["hoph_kprime"])
    flat = og.flat_layout(V, p["k"], p["kprime"])
    so, sh = og.oph_build_sketches(og.SetCollection.from_numpy(w.offsets, w.ids), V, seed, flat=flat, hier=hier)
    qo, qh = og.oph_build_sketches(og.SetCollection.from_numpy(w.q_offsets, w.q_ids), V, seed, flat=flat,
                                   hier=hier)
    glay = oracle.hoph_layout(V, p["a"], p["b"], p["hoph_kprime"])
    F = oracle.oph_sketch(w.offsets, w.ids, V, p["k"], seed)
    _check_sketches_chunked(so, F)
    H = oracle.hoph_sketch(w.offsets, w.ids, V, glay, p["hoph_kprime"], seed)
    _check_sketches_chunked(sh, H)
    sample = [shard * 1000 + 3, 16383 - shard]
    QF = oracle.oph_sketch(w.q_offsets, w.q_ids, V, p["k"], seed)
    QH = oracle.hoph_sketch(w.q_offsets, w.q_ids, V, glay, p["hoph_kprime"], seed)
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    for m in ("full", "goph", "hoph"):
        if m == "hoph":
            hits = gpu_threshold_hits(m, qh, sh, layout=hier, strategy=og.OPH_STRATEGY_AUTO, capacity=1 << 24, **kw)
            want = oracle_records(m, QH[sample], H, kprime=p["hoph_kprime"], L=len(glay), **kw)
        else:
            hits = gpu_threshold_hits(m, qo, so, layout=flat, strategy=og.OPH_STRATEGY_AUTO, capacity=1 << 24, **kw)
            want = oracle_records(m, QF[sample], F, k=p["k"], kprime=p["kprime"], **kw)
        got = [(int(h["query"]), int(h["set_id"])) for h in hits if int(h["query"]) in set(sample)]
        assert got == [(sample[q], s) for q, s in oracle.threshold_list(want)], (shard, m)
