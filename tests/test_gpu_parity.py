"""Parity of the CUDA path (through the C-ABI) with the CPU oracle.

Bar (B.north_star): sketches, per-pair match / excluded-bin counts, groups
compared, verdicts, flags and returned IDs bit-exact; estimates within 1e-6
absolute.  Inputs: the seeded generators in workloads/ (the oracle never
sees a value the GPU produced)."""
import numpy as np
import pytest

import oracle
import paper_1805_11254_b200 as og
from workloads import make_csr, text_like, tiny

from gpu_helpers import (assert_records_equal, gpu_build, gpu_dense, gpu_threshold_hits, masks_from_values,
                         oracle_records, subview)

pytestmark = pytest.mark.gpu

E = oracle.EMPTY


@pytest.fixture(scope="module", autouse=True)
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    og.build()


# ----------------------------------------------------------------------------- worked examples
def test_paper_worked_examples_on_gpu(golden):
    """P:158 OPH and P:482 HOPH goldens (identity psi) and their estimates."""
    g, h = golden("oph_example.json"), golden("hoph_example.json")
    names = ["D1", "D2", "D3"]
    offs, ids = make_csr([g["sets"][n] for n in names])
    hier = og.oph_hier_layout_make(17, 1, 1, 2)
    _, so, sh = gpu_build(offs, ids, 17, 0, k=4, kprime=2, hier=hier, identity=True)
    F, H = so.numpy(), sh.numpy()
    for i, n in enumerate(names):
        assert [None if v == E else int(v) for v in F[i]] == g["sketch"][n]
        assert [None if v == E else int(v) for v in H[i]] == h["sketch"][n]
    lay = og.flat_layout(17, 4, 2)
    full = gpu_dense("full", so, so, layout=lay, t_num=1, t_den=2)
    assert full[0, 1]["estimate"] == 0.75 and full[0, 1]["n_mb"] == 3
    assert abs(full[0, 2]["estimate"] - 1 / 3) < 1e-7
    joint = gpu_dense("full", so, so, layout=lay, t_num=1, t_den=2, joint=True)
    assert joint[0, 2]["estimate"] == 0.25
    # HOPH estimator: with eps -> 0 no small-probability stop can fire; (D1, D2) reaches the last group
    hp = gpu_dense("hoph", sh, sh, layout=hier, t_num=1, t_den=2, eps=1e-300)
    assert hp[0, 1]["groups"] == 3 and hp[0, 1]["estimate"] == 0.625


# ----------------------------------------------------------------------------- tiny (configs[0])
@pytest.fixture(scope="module")
def tiny_run():
    w = tiny()
    p = w.params
    hier = og.oph_hier_layout_make(w.vocab_size, p["a"], p["b"], p["hoph_kprime"])
    sets, so, sh = gpu_build(w.offsets, w.ids, w.vocab_size, p["perm_seed"], k=p["k"], kprime=p["kprime"], hier=hier)
    qsets, qo, qh = gpu_build(w.q_offsets, w.q_ids, w.vocab_size, p["perm_seed"], k=p["k"], kprime=p["kprime"],
                              hier=hier)
    mw = og.minwise_build_sketches(sets, w.vocab_size, p["perm_seed"], p["mw_k"])
    qmw = og.minwise_build_sketches(qsets, w.vocab_size, p["perm_seed"], p["mw_k"])
    lay = oracle.hoph_layout(w.vocab_size, p["a"], p["b"], p["hoph_kprime"])
    orc = dict(
        F=oracle.oph_sketch(w.offsets, w.ids, w.vocab_size, p["k"], p["perm_seed"]),
        QF=oracle.oph_sketch(w.q_offsets, w.q_ids, w.vocab_size, p["k"], p["perm_seed"]),
        H=oracle.hoph_sketch(w.offsets, w.ids, w.vocab_size, lay, p["hoph_kprime"], p["perm_seed"]),
        QH=oracle.hoph_sketch(w.q_offsets, w.q_ids, w.vocab_size, lay, p["hoph_kprime"], p["perm_seed"]),
        MW=oracle.minwise_sketch(w.offsets, w.ids, w.vocab_size, p["mw_k"], p["perm_seed"]),
        QMW=oracle.minwise_sketch(w.q_offsets, w.q_ids, w.vocab_size, p["mw_k"], p["perm_seed"]),
        L=len(lay))
    return dict(w=w, p=p, hier=hier, so=so, sh=sh, qo=qo, qh=qh, mw=mw, qmw=qmw, orc=orc)


def test_tiny_sketches_bit_exact(tiny_run):
    r, o = tiny_run, tiny_run["orc"]
    assert (r["so"].numpy() == o["F"]).all()
    assert (r["qo"].numpy() == o["QF"]).all()
    assert (r["sh"].numpy() == o["H"]).all()
    assert (r["qh"].numpy() == o["QH"]).all()
    assert (r["so"].empty_numpy() == masks_from_values(o["F"])).all()
    assert (r["sh"].empty_numpy() == masks_from_values(o["H"])).all()
    mw, fl = o["MW"]
    assert (r["mw"].numpy() == mw).all()
    assert (r["mw"].flags.cpu().numpy()[: len(fl)] == fl).all()


@pytest.mark.parametrize("strategy", [og.OPH_STRATEGY_BRUTE, og.OPH_STRATEGY_BITMAP])
@pytest.mark.parametrize("joint", [False, True])
@pytest.mark.parametrize("method", ["full", "goph", "hoph", "minwise"])
def test_tiny_dense_records(tiny_run, method, joint, strategy):
    r, o, p = tiny_run, tiny_run["orc"], tiny_run["p"]
    if method == "minwise" and (joint or strategy == og.OPH_STRATEGY_BITMAP):
        pytest.skip("MinWise has no empty bins / no BITMAP join")
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"], joint=joint, strategy=strategy)
    if method in ("full", "goph"):
        lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
        g = gpu_dense(method, r["qo"], r["so"], layout=lay, **kw)
        kw.pop("strategy")
        want = oracle_records(method, o["QF"], o["F"], k=p["k"], kprime=p["kprime"], **kw)
    elif method == "hoph":
        g = gpu_dense(method, r["qh"], r["sh"], layout=r["hier"], **kw)
        kw.pop("strategy")
        want = oracle_records(method, o["QH"], o["H"], kprime=p["hoph_kprime"], L=o["L"], **kw)
    else:
        g = gpu_dense(method, r["qmw"], r["mw"], **kw)
        kw.pop("strategy")
        want = oracle_records(method, o["QMW"][0], o["MW"][0], qflags=o["QMW"][1], sflags=o["MW"][1], **kw)
    assert_records_equal(g, want, f"tiny {method} joint={joint} strategy={strategy}")


@pytest.mark.parametrize("strategy", [og.OPH_STRATEGY_BRUTE, og.OPH_STRATEGY_PROBE, og.OPH_STRATEGY_BITMAP])
@pytest.mark.parametrize("method", ["full", "goph", "hoph", "minwise"])
def test_tiny_threshold_lists(tiny_run, method, strategy):
    """Threshold hit lists (sorted by (query, set_id)) == oracle's, with set_id_base, for every scan strategy."""
    r, o, p = tiny_run, tiny_run["orc"], tiny_run["p"]
    if method == "minwise" and strategy == og.OPH_STRATEGY_BITMAP:
        pytest.skip("no BITMAP join for MinWise")
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    base = 1000
    if method in ("full", "goph"):
        lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
        hits = gpu_threshold_hits(method, r["qo"], r["so"], layout=lay, set_id_base=base, strategy=strategy, **kw)
        want = oracle_records(method, o["QF"], o["F"], k=p["k"], kprime=p["kprime"], **kw)
    elif method == "hoph":
        hits = gpu_threshold_hits(method, r["qh"], r["sh"], layout=r["hier"], set_id_base=base, strategy=strategy, **kw)
        want = oracle_records(method, o["QH"], o["H"], kprime=p["hoph_kprime"], L=o["L"], **kw)
    else:
        hits = gpu_threshold_hits(method, r["qmw"], r["mw"], set_id_base=base, strategy=strategy, **kw)
        want = oracle_records(method, o["QMW"][0], o["MW"][0], qflags=o["QMW"][1], sflags=o["MW"][1], **kw)
    got = [(int(h["query"]), int(h["set_id"])) for h in hits]
    assert got == oracle.threshold_list(want, base)
    assert len(got) > 0
    # the records themselves match the dense oracle records
    for h in hits[:200]:
        wr = want[h["query"], h["set_id"] - base]
        assert (h["n_mb"], h["n_excl"], h["groups"], h["flags"]) == (wr["n_mb"], wr["n_excl"], wr["groups"], wr["flags"])


@pytest.mark.parametrize("nq", [1, 3, 4, 5, 8, 9, 16, 17, 33])
@pytest.mark.parametrize("method", ["full", "goph", "hoph", "minwise"])
def test_tiny_query_blocks(tiny_run, method, nq):
    """Dense records for 1 .. 33 queries: every register query block of the BRUTE
    scan (4 / 8 / 16 / 32 queries, the 4- and 8-query blocks at 8 / 7 CTAs per SM)
    and its partial last block; 33 adds a second 32-query block of one query."""
    r, o, p = tiny_run, tiny_run["orc"], tiny_run["p"]
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"], strategy=og.OPH_STRATEGY_BRUTE)
    if method in ("full", "goph"):
        lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
        g = gpu_dense(method, subview(r["qo"], nq), r["so"], layout=lay, **kw)
        want = oracle_records(method, o["QF"][:nq], o["F"], k=p["k"], kprime=p["kprime"], **kw)
    elif method == "hoph":
        g = gpu_dense(method, subview(r["qh"], nq), r["sh"], layout=r["hier"], **kw)
        want = oracle_records(method, o["QH"][:nq], o["H"], kprime=p["hoph_kprime"], L=o["L"], **kw)
    else:
        g = gpu_dense(method, subview(r["qmw"], nq), r["mw"], **kw)
        want = oracle_records(method, o["QMW"][0][:nq], o["MW"][0], qflags=o["QMW"][1][:nq], sflags=o["MW"][1], **kw)
    assert_records_equal(g, want, f"tiny {method} nq={nq}")


# ----------------------------------------------------------------------------- empty-aware GOPH (E1-E4)
@pytest.mark.parametrize("joint", [False, True])
def test_tiny_goph_empty_aware(tiny_run, joint):
    """The empty-aware GOPH rule (OPH_VARIANT_EMPTY_AWARE): dense records,
    threshold list and termination histogram == the oracle's (O9e)."""
    r, o, p = tiny_run, tiny_run["orc"], tiny_run["p"]
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"], joint=joint)
    lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
    want = oracle_records("goph_e", o["QF"], o["F"], k=p["k"], kprime=p["kprime"], **kw)
    g = gpu_dense("goph_e", r["qo"], r["so"], layout=lay, **kw)
    assert_records_equal(g, want, f"tiny goph_e joint={joint}")
    hits = gpu_threshold_hits("goph_e", r["qo"], r["so"], layout=lay, set_id_base=7, **kw)
    assert [(int(h["query"]), int(h["set_id"])) for h in hits] == oracle.threshold_list(want, 7)
    res = og.Results(1 << 20, stop_hist=True)
    og.compare_goph(r["qo"], r["so"], lay, og.params(p["t_num"], p["t_den"], p["eps"], joint,
                                                     variant=og.OPH_VARIANT_EMPTY_AWARE), res)
    assert np.array_equal(res.hist()[: p["k"] // p["kprime"] + 1],
                          np.bincount(want["groups"].ravel(), minlength=p["k"] // p["kprime"] + 1))
    # the variant finds at least the planted near-duplicates the paper rule finds
    paper = oracle_records("goph", o["QF"], o["F"], k=p["k"], kprime=p["kprime"], **kw)
    assert want["verdict"].sum() >= paper["verdict"].sum()


@pytest.mark.parametrize("V,k,kp,seed", [(1000003, 48, 16, 3), (4097, 96, 32, 4), (1 << 20, 512, 32, 5),
                                         (300, 30, 10, 6), (2, 1, 1, 8)])
def test_goph_empty_aware_ragged(V, k, kp, seed):
    """Ragged shapes for the variant: k not a multiple of 32, k' = 10, empty
    sets, a set and query count that are not multiples of a tile / block,
    many empty bins (sets of 0-60 ids); T = 1/2, eps = 1e-3."""
    rng = np.random.default_rng(seed)
    nset, nq = 517, 45
    sets_l = [np.sort(rng.choice(V, size=min(V, int(rng.integers(0, 60))), replace=False)) for _ in range(nset)]
    qs_l = [np.sort(rng.choice(V, size=min(V, int(rng.integers(0, 60))), replace=False)) for _ in range(nq)]
    for i in range(0, nq, 3):  # near-duplicates so some pairs reach late groups
        qs_l[i] = sets_l[i * 7 % nset]
    offs, ids = make_csr(sets_l)
    qoffs, qids = make_csr(qs_l)
    _, so, _ = gpu_build(offs, ids, V, seed, k=k, kprime=kp)
    _, qo, _ = gpu_build(qoffs, qids, V, seed, k=k, kprime=kp)
    F = oracle.oph_sketch(offs, ids, V, k, seed)
    QF = oracle.oph_sketch(qoffs, qids, V, k, seed)
    lay = og.flat_layout(V, k, kp)
    for joint in (False, True):
        kw = dict(t_num=1, t_den=2, eps=1e-3, joint=joint)
        want = oracle_records("goph_e", QF, F, k=k, kprime=kp, **kw)
        assert_records_equal(gpu_dense("goph_e", qo, so, layout=lay, **kw), want, f"goph_e V={V} k={k} joint={joint}")
        # threshold lists through the join + listed-pair path (E5) and through the register scan
        for strategy in (og.OPH_STRATEGY_PROBE, og.OPH_STRATEGY_BRUTE):
            hits = gpu_threshold_hits("goph_e", qo, so, layout=lay, strategy=strategy, **kw)
            assert [(int(h["query"]), int(h["set_id"])) for h in hits] == oracle.threshold_list(want)
            for h in hits:
                wr = want[h["query"], h["set_id"]]
                assert (h["n_mb"], h["n_excl"], h["groups"], h["flags"]) == \
                    (wr["n_mb"], wr["n_excl"], wr["groups"], wr["flags"])


def test_goph_empty_aware_invalid(tiny_run):
    """The variant is a GOPH / HOPH rule: full OPH (and MinWise) refuse it, and so does a GOPH
    layout with n k' > 512 (the register scan holds every group)."""
    r, p = tiny_run, tiny_run["p"]
    prm = og.params(p["t_num"], p["t_den"], p["eps"], variant=og.OPH_VARIANT_EMPTY_AWARE)
    lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
    with pytest.raises(RuntimeError):
        og.compare_full(r["qo"], r["so"], lay, prm, og.Results(1 << 16))
    with pytest.raises(RuntimeError):
        og.compare_minwise(r["qmw"], r["mw"], prm, og.Results(1 << 16))
    w = text_like(seed=3, n_sets=300, n_queries=10)
    big = og.flat_layout(w.vocab_size, 1024, 32)
    _, so, _ = gpu_build(w.offsets, w.ids, w.vocab_size, 1, k=1024, kprime=32)
    _, qo, _ = gpu_build(w.q_offsets, w.q_ids, w.vocab_size, 1, k=1024, kprime=32)
    with pytest.raises(RuntimeError):
        og.compare_goph(qo, so, big, prm, og.Results(1 << 16))


@pytest.mark.parametrize("method", ["full", "minwise"])
def test_tiny_topk(tiny_run, method):
    r, o, p = tiny_run, tiny_run["orc"], tiny_run["p"]
    kw = dict(t_num=1, t_den=10)
    if method == "full":
        lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
        res = og.Results(1 << 20)
        og.compare_full(r["qo"], r["so"], lay, og.params(1, 10, 1e-4), res)
        want = oracle_records(method, o["QF"], o["F"], k=p["k"], kprime=p["kprime"], **kw)
    else:
        res = og.Results(1 << 20)
        og.compare_minwise(r["qmw"], r["mw"], og.params(1, 10, 1e-4), res)
        want = oracle_records(method, o["QMW"][0], o["MW"][0], qflags=o["QMW"][1], sflags=o["MW"][1], **kw)
    n = res.n()
    out = og.Results(n)
    og.topk_or_threshold_results(res, n, og.OPH_SELECT_TOPK, out, topk=7, k_bins=p["k"])
    m = out.n()
    got = [(int(h["query"]), int(h["set_id"])) for h in out.numpy(m)]
    assert got == oracle.topk_list(want, p["k"], 7)


def test_tiny_query_chunking(tiny_run):
    """A survivor capacity of 32 * n_sets forces 4 query chunks: same records."""
    r, o, p = tiny_run, tiny_run["orc"], tiny_run["p"]
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    n_s = r["sh"].n_sets
    g = gpu_dense("hoph", r["qh"], r["sh"], layout=r["hier"], survivor_capacity=32 * n_s, **kw)
    want = oracle_records("hoph", o["QH"], o["H"], kprime=p["hoph_kprime"], L=o["L"], **kw)
    assert_records_equal(g, want, "tiny hoph chunked")


# ----------------------------------------------------------------------------- ragged / edge cases
@pytest.mark.parametrize("V,k,kp,hkp,seed", [(1000003, 48, 16, 8, 3), (4097, 96, 32, 32, 4), (1 << 20, 512, 32, 32, 5),
                                             (300, 30, 10, 5, 6), (1 << 32, 256, 32, 32, 7), (2, 1, 1, 1, 8)])
def test_ragged_and_edges(V, k, kp, hkp, seed):
    """Non-power-of-two |V| (cycle walking, exact division path), k not a
    multiple of 32, empty sets, n_sets and n_queries not multiples of the
    tile / query block, sets covering the whole universe."""
    rng = np.random.default_rng(seed)
    nset, nq = 517, 45
    sizes = rng.integers(0, 60, size=nset)
    sizes[:3] = 0
    sets = [rng.choice(V, size=min(int(s), V), replace=False) if s else [] for s in sizes]
    if V <= 4097:
        sets[3] = np.arange(V)
    qsets = [sets[i] if i % 3 == 0 else rng.choice(V, size=min(V, int(rng.integers(0, 60))), replace=False)
             for i in range(nq)]
    qsets[1] = []
    offs, ids = make_csr(sets)
    qoffs, qids = make_csr(qsets)
    hier = og.oph_hier_layout_make(V, 1, 1, hkp) if V >= 2 * hkp else None
    _, so, sh = gpu_build(offs, ids, V, seed, k=k, kprime=kp, hier=hier)
    _, qo, qh = gpu_build(qoffs, qids, V, seed, k=k, kprime=kp, hier=hier)
    F = oracle.oph_sketch(offs, ids, V, k, seed)
    QF = oracle.oph_sketch(qoffs, qids, V, k, seed)
    assert (so.numpy() == F).all() and (qo.numpy() == QF).all()
    assert (so.empty_numpy() == masks_from_values(F)).all()
    lay = og.flat_layout(V, k, kp)
    def strategies(kp_levels):  # BRUTE always; BITMAP where its domain allows (|V| <= 2^23, k' % 16)
        return (og.OPH_STRATEGY_BRUTE,) + ((og.OPH_STRATEGY_BITMAP,) if V <= (1 << 23) and kp_levels else ())
    for joint in (False, True):
        for st in strategies(True):
            kw = dict(t_num=7, t_den=10, eps=1e-4, joint=joint, strategy=st)
            assert_records_equal(gpu_dense("full", qo, so, layout=lay, **kw),
                                 oracle_records("full", QF, F, k=k, kprime=kp, **kw), f"full {V} {st}")
        for st in strategies(kp % 16 == 0):
            kw = dict(t_num=7, t_den=10, eps=1e-4, joint=joint, strategy=st)
            assert_records_equal(gpu_dense("goph", qo, so, layout=lay, **kw),
                                 oracle_records("goph", QF, F, k=k, kprime=kp, **kw), f"goph {V} {st}")
    if hier is not None:
        glay = oracle.hoph_layout(V, 1, 1, hkp)
        H = oracle.hoph_sketch(offs, ids, V, glay, hkp, seed)
        QH = oracle.hoph_sketch(qoffs, qids, V, glay, hkp, seed)
        assert (sh.numpy() == H).all() and (sh.empty_numpy() == masks_from_values(H)).all()
        hier_l = len(oracle.hoph_layout(V, 1, 1, hkp))
        for joint in (False, True):
            for st in strategies(hkp % 16 == 0 and 2 <= hier_l <= 20):
                kw = dict(t_num=7, t_den=10, eps=1e-4, joint=joint, strategy=st)
                assert_records_equal(gpu_dense("hoph", qh, sh, layout=hier, **kw),
                                     oracle_records("hoph", QH, H, kprime=hkp, L=len(glay), **kw), f"hoph {V} {st}")
    sets_t = og.SetCollection.from_numpy(offs, ids)
    q_t = og.SetCollection.from_numpy(qoffs, qids)
    mk = min(k, 64)
    mw = og.minwise_build_sketches(sets_t, V, seed, mk)
    qmw = og.minwise_build_sketches(q_t, V, seed, mk)
    MW, fl = oracle.minwise_sketch(offs, ids, V, mk, seed)
    QMW, qfl = oracle.minwise_sketch(qoffs, qids, V, mk, seed)
    assert (mw.numpy() == MW).all()
    assert_records_equal(gpu_dense("minwise", qmw, mw, t_num=7, t_den=10),
                         oracle_records("minwise", QMW, MW, qflags=qfl, sflags=fl, t_num=7, t_den=10), "minwise")


@pytest.mark.parametrize("tn,td,eps", [(1, 1, 1e-4), (1, 20, 1e-4), (7, 10, 0.5), (7, 10, 1e-300), (4, 5, 1e-2)])
@pytest.mark.parametrize("strategy", [og.OPH_STRATEGY_BRUTE, og.OPH_STRATEGY_BITMAP])
def test_threshold_and_epsilon_extremes(tiny_run, tn, td, eps, strategy):
    r, o, p = tiny_run, tiny_run["orc"], tiny_run["p"]
    kw = dict(t_num=tn, t_den=td, eps=eps, strategy=strategy)
    lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
    q = subview(r["qo"], 40)
    assert_records_equal(gpu_dense("goph", q, r["so"], layout=lay, **kw),
                         oracle_records("goph", o["QF"][:40], o["F"], k=p["k"], kprime=p["kprime"], **kw), "goph")
    qh = subview(r["qh"], 40)
    assert_records_equal(gpu_dense("hoph", qh, r["sh"], layout=r["hier"], **kw),
                         oracle_records("hoph", o["QH"][:40], o["H"], kprime=p["hoph_kprime"], L=o["L"], **kw), "hoph")


@pytest.mark.parametrize("method", ["full", "goph", "hoph", "minwise", "goph_e"])
def test_probe_overflow_falls_back_to_brute(method):
    """40 identical queries (plus 20 others): every set near them matches more
    than 4 distinct queries, so PROBE hands those sets to the BRUTE list
    scan; the hit lists still equal the oracle's."""
    rng = np.random.default_rng(12)
    V = 1 << 20
    A = rng.choice(V, size=300, replace=False)
    sets = []
    for i in range(700):
        if i % 7 == 0:  # near-duplicates of A
            keep = rng.choice(A, size=int(rng.integers(200, 300)), replace=False)
            sets.append(np.concatenate([keep, rng.choice(V, size=300 - len(keep), replace=False)]))
        else:
            sets.append(rng.choice(V, size=int(rng.integers(100, 400)), replace=False))
    qsets = [A] * 40 + [rng.choice(V, size=250, replace=False) for _ in range(20)]
    offs, ids = make_csr(sets)
    qoffs, qids = make_csr(qsets)
    hier = og.oph_hier_layout_make(V, 1, 1, 32)
    k, kp = 256, 32
    _, so, sh = gpu_build(offs, ids, V, 9, k=k, kprime=kp, hier=hier)
    _, qo, qh = gpu_build(qoffs, qids, V, 9, k=k, kprime=kp, hier=hier)
    kw = dict(t_num=3, t_den=5, eps=1e-4)
    lay = og.flat_layout(V, k, kp)
    if method == "hoph":
        glay = oracle.hoph_layout(V, 1, 1, 32)
        H = oracle.hoph_sketch(offs, ids, V, glay, 32, 9)
        QH = oracle.hoph_sketch(qoffs, qids, V, glay, 32, 9)
        want = oracle_records(method, QH, H, kprime=32, L=len(glay), **kw)
        hits = gpu_threshold_hits(method, qh, sh, layout=hier, strategy=og.OPH_STRATEGY_PROBE, **kw)
    elif method == "minwise":
        st, qt = og.SetCollection.from_numpy(offs, ids), og.SetCollection.from_numpy(qoffs, qids)
        mw, qmw = og.minwise_build_sketches(st, V, 9, 128), og.minwise_build_sketches(qt, V, 9, 128)
        MW, fl = oracle.minwise_sketch(offs, ids, V, 128, 9)
        QMW, qfl = oracle.minwise_sketch(qoffs, qids, V, 128, 9)
        want = oracle_records(method, QMW, MW, qflags=qfl, sflags=fl, **kw)
        hits = gpu_threshold_hits(method, qmw, mw, strategy=og.OPH_STRATEGY_PROBE, **kw)
    else:
        F = oracle.oph_sketch(offs, ids, V, k, 9)
        QF = oracle.oph_sketch(qoffs, qids, V, k, 9)
        want = oracle_records(method, QF, F, k=k, kprime=kp, **kw)
        hits = gpu_threshold_hits(method, qo, so, layout=lay, strategy=og.OPH_STRATEGY_PROBE, **kw)
    got = [(int(h["query"]), int(h["set_id"])) for h in hits]
    assert got == oracle.threshold_list(want)
    assert len(got) >= 40 * 50
    for h in hits[:500]:
        wr = want[h["query"], h["set_id"]]
        assert (h["n_mb"], h["n_excl"], h["groups"], h["flags"]) == (wr["n_mb"], wr["n_excl"], wr["groups"], wr["flags"])


@pytest.mark.parametrize("similar", [False, True])
def test_auto_decision_cache(similar):
    """AUTO samples the first 1/16 of a > 16,384-set collection once and remembers its
    decision for the buffer: the first call, the repeated calls (cached probe -> one join
    over every set; cached BRUTE -> BRUTE outright) and explicit BRUTE / PROBE return the
    same hit lists, equal to the oracle's for the sampled queries.  `similar`: every set
    shares most of its ids with the queries (the sample overflows the join's lists)."""
    rng = np.random.default_rng(77 + similar)
    V, k, kp, n_sets, nq = 1 << 20, 64, 16, 40_000, 40
    base = [rng.choice(V, size=80, replace=False) for _ in range(4)]
    sets_l = []
    for i in range(n_sets):
        if similar:
            b = base[i % 4]
            keep = b[rng.random(80) < 0.85]
            sets_l.append(np.unique(np.concatenate([keep, rng.choice(V, size=10, replace=False)])))
        else:
            sets_l.append(np.unique(rng.choice(V, size=int(rng.integers(40, 120)), replace=False)))
    qs_l = [base[i % 4] if similar else sets_l[i * 997 % n_sets] for i in range(nq)]
    offs, ids = make_csr(sets_l)
    qoffs, qids = make_csr([np.sort(q) for q in qs_l])
    _, so, sh = gpu_build(offs, ids, V, 5, k=k, kprime=kp)
    _, qo, _ = gpu_build(qoffs, qids, V, 5, k=k, kprime=kp)
    lay = og.flat_layout(V, k, kp)
    kw = dict(t_num=7, t_den=10, eps=1e-4)
    for method in ("full", "goph"):
        runs = [gpu_threshold_hits(method, qo, so, layout=lay, strategy=st, capacity=1 << 22,
                                   survivor_capacity=32 * n_sets, **kw)
                for st in (og.OPH_STRATEGY_AUTO, og.OPH_STRATEGY_AUTO, og.OPH_STRATEGY_AUTO,
                           og.OPH_STRATEGY_BRUTE, og.OPH_STRATEGY_PROBE)]
        lists = [[(int(h["query"]), int(h["set_id"])) for h in r] for r in runs]
        assert all(x == lists[0] for x in lists[1:]), method
        F = oracle.oph_sketch(offs, ids, V, k, 5)
        QF = oracle.oph_sketch(qoffs, qids, V, k, 5)
        want = oracle_records(method, QF[:2], F, k=k, kprime=kp, **kw)
        assert [x for x in lists[0] if x[0] < 2] == oracle.threshold_list(want)
        assert len(lists[0]) > 0


@pytest.mark.parametrize("a,b,V,kp", [(1, 2, 1 << 20, 32), (2, 1, 1 << 20, 32), (3, 1, 1 << 16, 16), (1, 1, 100003, 16),
                                      (1, 2, 1 << 32, 32), (2, 1, 1 << 32, 32)])
def test_hoph_split_ratios(a, b, V, kp):
    """(a:b)HOPH variants of P:801-803 (general nominal weights, binary-search
    group lookup): sketches and dense records bit-exact, both empty modes.  At
    |V| = 2^32 the 1:2 split has L = 45 groups and weights up to 3^44, so the
    pair state S_l needs 128 bits; its threshold lists are
    checked for both scan strategies too."""
    rng = np.random.default_rng(a * 10 + b + (V >> 31))

    def draw(n):
        if V <= 1 << 24:
            return rng.choice(V, size=n, replace=False)
        return np.unique(rng.integers(0, V, size=n, dtype=np.uint64))

    sets = [draw(int(rng.integers(0, 700))) for _ in range(300)]
    qsets = [sets[i] if i % 2 == 0 else draw(400) for i in range(40)]
    offs, ids = make_csr(sets)
    qoffs, qids = make_csr(qsets)
    hier = og.oph_hier_layout_make(V, a, b, kp)
    glay = oracle.hoph_layout(V, a, b, kp)
    assert hier.groups() == glay
    _, _, sh = gpu_build(offs, ids, V, 21, hier=hier)
    _, _, qh = gpu_build(qoffs, qids, V, 21, hier=hier)
    H = oracle.hoph_sketch(offs, ids, V, glay, kp, 21)
    QH = oracle.hoph_sketch(qoffs, qids, V, glay, kp, 21)
    assert (sh.numpy() == H).all() and (qh.numpy() == QH).all()
    for joint in (False, True):
        kw = dict(t_num=3, t_den=5, eps=1e-4, joint=joint)
        want = oracle_records("hoph", QH, H, kprime=kp, L=len(glay), a=a, b=b, **kw)
        assert_records_equal(gpu_dense("hoph", qh, sh, layout=hier, **kw), want, f"hoph {a}:{b}")
        if V == 1 << 32:
            for strategy in (og.OPH_STRATEGY_BRUTE, og.OPH_STRATEGY_PROBE):
                hits = gpu_threshold_hits("hoph", qh, sh, layout=hier, strategy=strategy, **kw)
                assert [(int(h["query"]), int(h["set_id"])) for h in hits] == oracle.threshold_list(want, 0)


def test_empty_inputs():
    """Zero queries or zero sets: nothing is written, no error."""
    offs, ids = make_csr([[1, 2, 3]])
    e_offs, e_ids = make_csr([])
    _, so, _ = gpu_build(offs, ids, 1 << 16, 1, k=64, kprime=16)
    res = og.Results(10)
    lay = og.flat_layout(1 << 16, 64, 16)
    q0 = subview(so, 0)
    og.compare_full(q0, so, lay, og.params(7, 10, 1e-4), res)
    og.compare_goph(so, q0, lay, og.params(7, 10, 1e-4), res)
    assert res.n() == 0


# ----------------------------------------------------------------------------- text-like (configs[1]) at full size
@pytest.fixture(scope="module")
def text_run():
    w = text_like()
    p = w.params
    hier = og.oph_hier_layout_make(w.vocab_size, 1, 1, p["hoph_kprime"])
    sets, so, sh = gpu_build(w.offsets, w.ids, w.vocab_size, p["perm_seed"], k=p["k"], kprime=p["kprime"], hier=hier)
    qsets, qo, qh = gpu_build(w.q_offsets, w.q_ids, w.vocab_size, p["perm_seed"], k=p["k"], kprime=p["kprime"],
                              hier=hier)
    lay = oracle.hoph_layout(w.vocab_size, 1, 1, p["hoph_kprime"])
    return dict(w=w, p=p, hier=hier, sets=sets, so=so, sh=sh, qsets=qsets, qo=qo, qh=qh, glay=lay)


def test_text_sketches_full_collection(text_run):
    r = text_run
    w, p = r["w"], r["p"]
    F = oracle.oph_sketch(w.offsets, w.ids, w.vocab_size, p["k"], p["perm_seed"])
    assert (r["so"].numpy() == F).all()
    assert (r["so"].empty_numpy() == masks_from_values(F)).all()
    H = oracle.hoph_sketch(w.offsets, w.ids, w.vocab_size, r["glay"], p["hoph_kprime"], p["perm_seed"])
    assert (r["sh"].numpy() == H).all()
    r["F"], r["H"] = F, H


@pytest.mark.parametrize("method", ["full", "goph", "hoph"])
def test_text_all_queries_hit_lists(text_run, method):
    """configs[1] as the bench runs it (AUTO: the PROBE join): the hit lists of ALL 1,000
    queries x 200,000 sets, every record field, == the oracle's (evaluated in query chunks)."""
    r = text_run
    w, p = r["w"], r["p"]
    if "F" not in r:
        r["F"] = oracle.oph_sketch(w.offsets, w.ids, w.vocab_size, p["k"], p["perm_seed"])
        r["H"] = oracle.hoph_sketch(w.offsets, w.ids, w.vocab_size, r["glay"], p["hoph_kprime"], p["perm_seed"])
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    if method == "hoph":
        Q = oracle.hoph_sketch(w.q_offsets, w.q_ids, w.vocab_size, r["glay"], p["hoph_kprime"], p["perm_seed"])
        hits = gpu_threshold_hits(method, r["qh"], r["sh"], layout=r["hier"], strategy=og.OPH_STRATEGY_AUTO, **kw)
    else:
        Q = oracle.oph_sketch(w.q_offsets, w.q_ids, w.vocab_size, p["k"], p["perm_seed"])
        lay = og.flat_layout(w.vocab_size, p["k"], p["kprime"])
        hits = gpu_threshold_hits(method, r["qo"], r["so"], layout=lay, strategy=og.OPH_STRATEGY_AUTO, **kw)
    want = []
    rec = {}
    for q0 in range(0, Q.shape[0], 50):
        if method == "hoph":
            o = oracle_records(method, Q[q0:q0 + 50], r["H"], kprime=p["hoph_kprime"], L=len(r["glay"]), **kw)
        else:
            o = oracle_records(method, Q[q0:q0 + 50], r["F"], k=p["k"], kprime=p["kprime"], **kw)
        for q, s in oracle.threshold_list(o):
            want.append((q0 + q, s))
            rec[(q0 + q, s)] = o[q, s]
    got = [(int(h["query"]), int(h["set_id"])) for h in hits]
    assert got == want
    assert len(want) > 500
    for h in hits:
        o = rec[(int(h["query"]), int(h["set_id"]))]
        assert (h["n_mb"], h["n_excl"], h["groups"], h["flags"]) == (o["n_mb"], o["n_excl"], o["groups"], o["flags"])


@pytest.mark.parametrize("strategy", [og.OPH_STRATEGY_AUTO, og.OPH_STRATEGY_BRUTE])
@pytest.mark.parametrize("method", ["full", "goph", "hoph", "goph_e"])
def test_text_full_size_sampled_queries(text_run, method, strategy):
    """All 1,000 queries x 200,000 sets in the bench launch configuration
    (threshold mode); the hit lists of 8 sampled queries == the oracle's, and
    dense records of those 8 queries x all sets are bit-exact."""
    r = text_run
    w, p = r["w"], r["p"]
    if "F" not in r:
        r["F"] = oracle.oph_sketch(w.offsets, w.ids, w.vocab_size, p["k"], p["perm_seed"])
        r["H"] = oracle.hoph_sketch(w.offsets, w.ids, w.vocab_size, r["glay"], p["hoph_kprime"], p["perm_seed"])
    sample = [0, 1, 7, 100, 333, 500, 998, 999]
    qo_np = oracle.oph_sketch(w.q_offsets, w.q_ids, w.vocab_size, p["k"], p["perm_seed"])
    qh_np = oracle.hoph_sketch(w.q_offsets, w.q_ids, w.vocab_size, r["glay"], p["hoph_kprime"], p["perm_seed"])
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    lay = og.flat_layout(w.vocab_size, p["k"], p["kprime"])
    if method == "hoph":
        hits = gpu_threshold_hits(method, r["qh"], r["sh"], layout=r["hier"], strategy=strategy, **kw)
        want = oracle_records(method, qh_np[sample], r["H"], kprime=p["hoph_kprime"], L=len(r["glay"]), **kw)
    else:
        hits = gpu_threshold_hits(method, r["qo"], r["so"], layout=lay, strategy=strategy, **kw)
        want = oracle_records(method, qo_np[sample], r["F"], k=p["k"], kprime=p["kprime"], **kw)
    got = [(int(h["query"]), int(h["set_id"])) for h in hits if int(h["query"]) in sample]
    exp = [(sample[q], s) for q, s in oracle.threshold_list(want)]
    assert got == exp
    # every planted duplicate of a sampled query with high J is found by full OPH
    if method == "full":
        planted = {(int(q), int(s)) for q, s, i, u in w.planted if q in sample and i / u >= 0.9}
        assert planted <= set(got)
    # dense records of the first sampled queries (a contiguous query subview)
    q8 = subview(r["qh"] if method == "hoph" else r["qo"], 8)
    if method == "hoph":
        g = gpu_dense(method, q8, r["sh"], layout=r["hier"], **kw)
        o8 = oracle_records(method, qh_np[:8], r["H"], kprime=p["hoph_kprime"], L=len(r["glay"]), **kw)
    else:
        g = gpu_dense(method, q8, r["so"], layout=lay, **kw)
        o8 = oracle_records(method, qo_np[:8], r["F"], k=p["k"], kprime=p["kprime"], **kw)
    assert_records_equal(g, o8, f"text {method}")


def test_text_minwise_subset(text_run):
    """MinWise sketches (sampled 20,000 sets) and scoring of 32 queries."""
    r = text_run
    w, p = r["w"], r["p"]
    n = 20_000
    offs = w.offsets[: n + 1]
    sets = og.SetCollection.from_numpy(offs, w.ids[: int(offs[-1])])
    mw = og.minwise_build_sketches(sets, w.vocab_size, p["perm_seed"], p["mw_k"])
    MW, fl = oracle.minwise_sketch(offs, w.ids, w.vocab_size, p["mw_k"], p["perm_seed"])
    assert (mw.numpy() == MW).all()
    qoffs = w.q_offsets[:33]
    qs = og.SetCollection.from_numpy(qoffs, w.q_ids[: int(qoffs[-1])])
    qmw = og.minwise_build_sketches(qs, w.vocab_size, p["perm_seed"], p["mw_k"])
    QMW, qfl = oracle.minwise_sketch(qoffs, w.q_ids, w.vocab_size, p["mw_k"], p["perm_seed"])
    kw = dict(t_num=p["t_num"], t_den=p["t_den"])
    assert_records_equal(gpu_dense("minwise", qmw, mw, **kw),
                         oracle_records("minwise", QMW, MW, qflags=qfl, sflags=fl, **kw), "text minwise")


# ----------------------------------------------------------------------------- PROBE filter widths / passes
@pytest.fixture(scope="module")
def wide_run():
    """6,000 text-like sets (30 % planted) and 5,000 queries: 1,500 queries make one
    PROBE pass with 1,024-word filters, 5,000 make two balanced passes of 2,528
    queries with 2,048-word filters (8-bin slabs)."""
    w = text_like(seed=11, n_sets=6000, n_queries=5000, planted_frac=0.3)
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    hier = og.oph_hier_layout_make(V, p["a"], p["b"], p["hoph_kprime"])
    _, so, sh = gpu_build(w.offsets, w.ids, V, seed, k=p["k"], kprime=p["kprime"], hier=hier)
    _, qo, qh = gpu_build(w.q_offsets, w.q_ids, V, seed, k=p["k"], kprime=p["kprime"], hier=hier)
    lay = oracle.hoph_layout(V, p["a"], p["b"], p["hoph_kprime"])
    return dict(w=w, p=p, hier=hier, so=so, sh=sh, qo=qo, qh=qh, L=len(lay),
                F=oracle.oph_sketch(w.offsets, w.ids, V, p["k"], seed),
                QF=oracle.oph_sketch(w.q_offsets, w.q_ids, V, p["k"], seed),
                H=oracle.hoph_sketch(w.offsets, w.ids, V, lay, p["hoph_kprime"], seed),
                QH=oracle.hoph_sketch(w.q_offsets, w.q_ids, V, lay, p["hoph_kprime"], seed))


@pytest.mark.parametrize("method,nq", [("full", 1500), ("goph", 1500), ("full", 5000), ("hoph", 5000)])
def test_probe_filter_widths(wide_run, method, nq):
    """PROBE threshold lists == oracle's for 1,024- and 2,048-word filters and multi-pass query batches."""
    r, p = wide_run, wide_run["p"]
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    if method == "hoph":
        q = subview(r["qh"], nq)
        hits = gpu_threshold_hits(method, q, r["sh"], layout=r["hier"], strategy=og.OPH_STRATEGY_PROBE,
                                  capacity=1 << 22, **kw)
        want = oracle_records(method, r["QH"][:nq], r["H"], kprime=p["hoph_kprime"], L=r["L"], **kw)
    else:
        lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
        q = subview(r["qo"], nq)
        hits = gpu_threshold_hits(method, q, r["so"], layout=lay, strategy=og.OPH_STRATEGY_PROBE,
                                  capacity=1 << 22, **kw)
        want = oracle_records(method, r["QF"][:nq], r["F"], k=p["k"], kprime=p["kprime"], **kw)
    got = [(int(h["query"]), int(h["set_id"])) for h in hits]
    assert got == oracle.threshold_list(want, 0)
    assert len(got) > 100
    for h in hits[:: max(1, len(hits) // 300)]:  # sampled records: counts and flags bit-exact
        o = want[int(h["query"]), int(h["set_id"])]
        assert (int(h["n_mb"]), int(h["n_excl"]), int(h["groups"]), int(h["verdict"]), int(h["flags"])) == \
            (int(o["n_mb"]), int(o["n_excl"]), int(o["groups"]), int(o["verdict"]), int(o["flags"]))


# ----------------------------------------------------------------------------- termination-level histograms
@pytest.mark.parametrize("strategy", [og.OPH_STRATEGY_BRUTE, og.OPH_STRATEGY_PROBE, og.OPH_STRATEGY_BITMAP])
@pytest.mark.parametrize("method", ["full", "goph", "hoph", "minwise"])
def test_tiny_stop_histogram(tiny_run, method, strategy):
    """d_stop_hist == the histogram of the oracle's per-pair `groups` (groups compared when
    decided: Alg. 1 / Alg. 2 early termination), summing to Q x N, for every scan strategy."""
    r, o, p = tiny_run, tiny_run["orc"], tiny_run["p"]
    if method == "minwise" and strategy == og.OPH_STRATEGY_BITMAP:
        pytest.skip("no BITMAP join for MinWise")
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    res = og.Results(1 << 20, stop_hist=True)
    prm = og.params(p["t_num"], p["t_den"], p["eps"], False, strategy)
    if method in ("full", "goph"):
        lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
        (og.compare_full if method == "full" else og.compare_goph)(r["qo"], r["so"], lay, prm, res)
        want = oracle_records(method, o["QF"], o["F"], k=p["k"], kprime=p["kprime"], **kw)
        q, s = r["qo"], r["so"]
    elif method == "hoph":
        og.compare_hoph(r["qh"], r["sh"], r["hier"], prm, res)
        want = oracle_records(method, o["QH"], o["H"], kprime=p["hoph_kprime"], L=o["L"], **kw)
        q, s = r["qh"], r["sh"]
    else:
        og.compare_minwise(r["qmw"], r["mw"], prm, res)
        want = oracle_records(method, o["QMW"][0], o["MW"][0], qflags=o["QMW"][1], sflags=o["MW"][1], **kw)
        q, s = r["qmw"], r["mw"]
    got = res.hist()
    exp = np.bincount(want["groups"].astype(np.int64).ravel(), minlength=og.OPH_STOP_HIST_LEN)
    assert int(got.sum()) == q.n_sets * s.n_sets
    assert (got.astype(np.int64) == exp).all(), (got[:20], exp[:20])
    if method in ("goph", "hoph"):  # early termination does save work on tiny
        assert exp[: (p["k"] // p["kprime"] if method == "goph" else o["L"])].sum() > 0


# ----------------------------------------------------------------------------- exact Jaccard verifier
def test_exact_jaccard_pairs_vs_oracle():
    """exact_jaccard_pairs: |A n B|, |A u B| bit-exact vs the oracle's sorted merge (O11, Eq. 5)
    for planted near-duplicates, random pairs, and empty / singleton / identical sets."""
    w = tiny()
    sets_l = [w.ids[int(w.offsets[i]):int(w.offsets[i + 1])] for i in range(w.n_sets)]
    qs_l = [w.q_ids[int(w.q_offsets[i]):int(w.q_offsets[i + 1])] for i in range(len(w.q_offsets) - 1)]
    sets_l += [np.zeros(0, np.uint32), np.array([5], np.uint32), qs_l[0]]   # empty, singleton, identical
    qs_l += [np.zeros(0, np.uint32)]                                        # empty query
    so, si = make_csr(sets_l)
    qo, qi = make_csr(qs_l)
    S = og.SetCollection.from_numpy(so, si)
    Qc = og.SetCollection.from_numpy(qo, qi)
    rng = np.random.default_rng(7)
    nq, ns = len(qs_l), len(sets_l)
    pairs = [(int(q), int(s)) for q, s, _, _ in w.planted]
    pairs += [(int(rng.integers(nq)), int(rng.integers(ns))) for _ in range(3000)]
    pairs += [(q, s) for q in (0, nq - 1) for s in (ns - 3, ns - 2, ns - 1)]
    import torch
    qa = torch.tensor([p[0] for p in pairs], dtype=torch.int32, device="cuda")
    sa = torch.tensor([p[1] for p in pairs], dtype=torch.int32, device="cuda")
    inter, union = og.exact_jaccard_pairs(Qc, S, qa, sa)
    inter, union = inter.cpu().numpy(), union.cpu().numpy()
    for i, (q, s) in enumerate(pairs):
        _, oi, ou = oracle.jaccard(qs_l[q], sets_l[s])
        assert (int(inter[i]), int(union[i])) == (oi, ou), (q, s)
    # the planted pairs carry their realised intersection / union (workloads: i = round(2sJ/(1+J)))
    for i, (q, s, pi, pu) in enumerate(w.planted):
        assert (int(inter[i]), int(union[i])) == (int(pi), int(pu))


# ----------------------------------------------------------------------------- parameter sweeps
@pytest.mark.parametrize("strategy", [og.OPH_STRATEGY_BRUTE, og.OPH_STRATEGY_BITMAP])
@pytest.mark.parametrize("kprime", [8, 16, 32])
@pytest.mark.parametrize("t_num,t_den", [(1, 2), (3, 5), (4, 5), (9, 10)])
@pytest.mark.parametrize("eps", [1e-3, 1e-5])
def test_tiny_parameter_sweep(tiny_run, kprime, t_num, t_den, eps, strategy):
    """The paper's sweeps (GOPH group count n = k/k', T in [0.5, 0.9], eps in {1e-3, 1e-5}):
    GOPH and HOPH dense records bit-exact with the oracle (tiny, k = 64), BRUTE and BITMAP."""
    r, o, p = tiny_run, tiny_run["orc"], tiny_run["p"]
    if strategy == og.OPH_STRATEGY_BITMAP and kprime % 16:
        pytest.skip("BITMAP levels are whole batches of 16 bins")
    w = r["w"]
    V = w.vocab_size
    kw = dict(t_num=t_num, t_den=t_den, eps=eps, strategy=strategy)
    lay = og.flat_layout(V, p["k"], kprime)
    assert_records_equal(gpu_dense("goph", r["qo"], r["so"], layout=lay, **kw),
                         oracle_records("goph", o["QF"], o["F"], k=p["k"], kprime=kprime, **kw),
                         f"goph k'={kprime} T={t_num}/{t_den} eps={eps}")
    hier = og.oph_hier_layout_make(V, 1, 1, kprime)
    glay = oracle.hoph_layout(V, 1, 1, kprime)
    seed = p["perm_seed"]
    _, _, sh = gpu_build(w.offsets, w.ids, V, seed, hier=hier)
    _, _, qh = gpu_build(w.q_offsets, w.q_ids, V, seed, hier=hier)
    H = oracle.hoph_sketch(w.offsets, w.ids, V, glay, kprime, seed)
    QH = oracle.hoph_sketch(w.q_offsets, w.q_ids, V, glay, kprime, seed)
    assert_records_equal(gpu_dense("hoph", qh, sh, layout=hier, **kw),
                         oracle_records("hoph", QH, H, kprime=kprime, L=len(glay), **kw),
                         f"hoph k'={kprime} T={t_num}/{t_den} eps={eps}")


# ----------------------------------------------------------------------------- shingling (ingestion)
def _synthetic_docs(rng, n_docs):
    words = [b"alpha", b"Beta", b"GAMMA", b"delta", b"eps", b"x", b"don't", b"e-mail", b"42", bytes([0xC3, 0xA9, 0x74])]
    seps = [b" ", b"  ", b"\t", b"\n", b"\r\n", b" \x0b ", b"\x0c"]
    docs = []
    for d in range(n_docs):
        n = int(rng.integers(0, 40)) if d % 7 else int(rng.integers(0, 3))  # some empty / short documents
        parts = []
        if rng.random() < 0.3:
            parts.append(seps[int(rng.integers(len(seps)))])                # leading whitespace
        for _ in range(n):
            parts.append(words[int(rng.integers(len(words)))])
            parts.append(seps[int(rng.integers(len(seps)))])
        docs.append(b"".join(parts))
    return docs


@pytest.mark.parametrize("w,V", [(1, 1 << 32), (3, 1 << 32), (5, 1 << 20), (2, 1000003)])
def test_shingle_text_vs_oracle(w, V):
    """GPU shingling == the oracle's CSR bit-exact (ids strictly increasing per document), and the
    result feeds the OPH build (end to end: text -> sets -> sketches == oracle sketches)."""
    import torch
    from oracle import shingle as osh
    rng = np.random.default_rng(w * 31 + (V & 0xFF))
    docs = _synthetic_docs(rng, 600)
    text = b"".join(docs)
    offs = np.zeros(len(docs) + 1, dtype=np.int64)
    np.cumsum([len(d) for d in docs], out=offs[1:])
    t = torch.from_numpy(np.frombuffer(text, dtype=np.uint8).copy()).cuda()
    o = torch.from_numpy(offs).cuda()
    sets = og.shingle_text(t, o, w, V, seed=1234)
    want_off, want_ids = osh.shingle_docs(docs, w, V, 1234)
    got_off = sets.offsets.cpu().numpy().astype(np.uint64)
    got_ids = sets.ids.cpu().numpy().view(np.uint32)
    assert (got_off == want_off).all()
    assert (got_ids == want_ids).all()
    assert want_off[-1] > 0
    if V >= 4096:
        hier = og.oph_hier_layout_make(V, 1, 1, 16)
        flat = og.flat_layout(V, 64, 16)
        so, _ = og.oph_build_sketches(sets, V, 9, flat=flat, hier=hier)
        assert (so.numpy() == oracle.oph_sketch(want_off, want_ids, V, 64, 9)).all()


@pytest.mark.parametrize("method", ["goph", "hoph"])
def test_tiny_survivor_path_dense(tiny_run, method, monkeypatch):
    """The BRUTE survivor-list path (first decidable level + level_kernel), which levels_kernel
    replaces whenever the states fit 32 bits, stays bit-exact: forced on tiny, dense records."""
    monkeypatch.setenv("OPHGPU_NO_MULTI_LEVEL_SCAN", "1")
    r, o, p = tiny_run, tiny_run["orc"], tiny_run["p"]
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    if method == "goph":
        lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
        g = gpu_dense("goph", r["qo"], r["so"], layout=lay, **kw)
        want = oracle_records("goph", o["QF"], o["F"], k=p["k"], kprime=p["kprime"], **kw)
    else:
        g = gpu_dense("hoph", r["qh"], r["sh"], layout=r["hier"], **kw)
        want = oracle_records("hoph", o["QH"], o["H"], kprime=p["hoph_kprime"], L=o["L"], **kw)
    assert_records_equal(g, want, f"tiny {method} survivor path")


def test_survivor_lists_many_late_pairs(monkeypatch):
    """Regression (ping-pong of the survivor lists): GOPH with the survivor-list path forced
    (OPHGPU_NO_MULTI_LEVEL_SCAN) on a collection whose pairs sit near T, so that far more
    than one grid stride of level_kernel (296 x 256 = 75,776 threads) survives past the
    first survivor launch (levels l0+1 .. l0+4).  The first launch must read one list and
    append to the other; hit list and termination histogram == the oracle's."""
    monkeypatch.setenv("OPHGPU_NO_MULTI_LEVEL_SCAN", "1")
    from workloads.gen import _uniform_sampler, plant_duplicate, sample_sets
    rng = np.random.default_rng(77)
    V, k, kp, tn, td, eps = 1 << 20, 512, 32, 7, 10, 1e-4
    draw = _uniform_sampler(V)
    _, hub = sample_sets(rng, np.array([800]), V, draw)
    qs = [plant_duplicate(rng, hub, 0.98, V, draw)[0] for _ in range(64)]
    ss = [plant_duplicate(rng, hub, float(rng.uniform(0.64, 0.86)), V, draw)[0] for _ in range(3000)]
    qo_, qi_ = make_csr(qs)
    so_, si_ = make_csr(ss)
    _, qo, _ = gpu_build(qo_, qi_, V, 5, k=k, kprime=kp)
    _, so, _ = gpu_build(so_, si_, V, 5, k=k, kprime=kp)
    lay = og.flat_layout(V, k, kp)
    l0 = og.plan_thresholds(og.OPH_METHOD_GOPH, k // kp, kp, tn, td, eps)[2]
    res = og.Results(1 << 20, stop_hist=True)
    og.compare_goph(qo, so, lay, og.params(tn, td, eps, strategy=og.OPH_STRATEGY_BRUTE), res,
                    survivor_capacity=64 * 3000)
    hist = res.hist().astype(np.int64)
    QF = oracle.oph_sketch(qo_, qi_, V, k, 5)
    F = oracle.oph_sketch(so_, si_, V, k, 5)
    want = oracle_records("goph", QF, F, t_num=tn, t_den=td, eps=eps, k=k, kprime=kp)
    assert hist[l0 + 5:].sum() > 75_776, hist  # the case the bug needs
    assert (hist == np.bincount(want["groups"].ravel(), minlength=len(hist))).all()
    n = res.n()
    out = og.Results(max(n, 1))
    og.topk_or_threshold_results(res, n, og.OPH_SELECT_THRESHOLD, out)
    got = out.numpy(n)
    wl = oracle.threshold_list(want)
    assert list(zip(got["query"].tolist(), got["set_id"].tolist())) == wl
    sel = want[got["query"].astype(np.int64), got["set_id"].astype(np.int64)]
    for f in ("n_mb", "n_excl", "groups", "verdict", "flags"):
        assert (got[f].astype(np.int64) == sel[f].astype(np.int64)).all(), f


# ----------------------------------------------------------------------------- BITMAP join (K7)
@pytest.fixture(scope="module")
def image_small():
    """An image-like collection (Zipf words over 2^20, k = 512, k' = 32, HOPH L = 15) with
    2,100 queries: two BITMAP query blocks of 2,048, the last one ragged (HOPH: group 1
    bit-sliced, the undecided pairs walked per pair over both query words of a lane)."""
    from workloads import gen
    w = gen.image_like(n_sets=20_000, n_queries=2100)
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    hier = og.oph_hier_layout_make(V, 1, 1, p["hoph_kprime"])
    _, so, sh = gpu_build(w.offsets, w.ids, V, seed, k=p["k"], kprime=p["kprime"], hier=hier)
    _, qo, qh = gpu_build(w.q_offsets, w.q_ids, V, seed, k=p["k"], kprime=p["kprime"], hier=hier)
    glay = oracle.hoph_layout(V, 1, 1, p["hoph_kprime"])
    orc = dict(F=oracle.oph_sketch(w.offsets, w.ids, V, p["k"], seed),
               QF=oracle.oph_sketch(w.q_offsets, w.q_ids, V, p["k"], seed),
               H=oracle.hoph_sketch(w.offsets, w.ids, V, glay, p["hoph_kprime"], seed),
               QH=oracle.hoph_sketch(w.q_offsets, w.q_ids, V, glay, p["hoph_kprime"], seed), L=len(glay))
    return dict(w=w, p=p, hier=hier, so=so, sh=sh, qo=qo, qh=qh, orc=orc)


@pytest.mark.parametrize("joint", [False, True])
@pytest.mark.parametrize("method", ["full", "goph", "hoph"])
def test_bitmap_image_like_dense(image_small, method, joint):
    """BITMAP dense records of all 2,100 queries x the first 2,000 sets == the oracle."""
    r, o, p = image_small, image_small["orc"], image_small["p"]
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"], joint=joint, strategy=og.OPH_STRATEGY_BITMAP)
    n = 2000
    if method == "hoph":
        g = gpu_dense(method, r["qh"], subview(r["sh"], n), layout=r["hier"], **kw)
        want = oracle_records(method, o["QH"], o["H"][:n], kprime=p["hoph_kprime"], L=o["L"], **kw)
    else:
        lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
        g = gpu_dense(method, r["qo"], subview(r["so"], n), layout=lay, **kw)
        want = oracle_records(method, o["QF"], o["F"][:n], k=p["k"], kprime=p["kprime"], **kw)
    assert_records_equal(g, want, f"bitmap image-like {method} joint={joint}")


@pytest.mark.parametrize("method", ["full", "goph", "hoph"])
def test_bitmap_image_like_lists_and_histogram(image_small, method):
    """BITMAP threshold lists (every record field) and termination histogram over all
    20,000 sets x 1,100 queries == the oracle's; equal to the BRUTE strategy's list."""
    r, o, p = image_small, image_small["orc"], image_small["p"]
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    if method == "hoph":
        q, s, lay = r["qh"], r["sh"], r["hier"]
        want = oracle_records(method, o["QH"], o["H"], kprime=p["hoph_kprime"], L=o["L"], **kw)
    else:
        q, s, lay = r["qo"], r["so"], og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
        want = oracle_records(method, o["QF"], o["F"], k=p["k"], kprime=p["kprime"], **kw)
    res = og.Results(1 << 22, stop_hist=True)
    prm = og.params(p["t_num"], p["t_den"], p["eps"], strategy=og.OPH_STRATEGY_BITMAP)
    fn = {"full": og.compare_full, "goph": og.compare_goph, "hoph": og.compare_hoph}[method]
    # a workspace full of garbage: nothing may rely on it being zero (r02: the zero row of the
    # 2,048-query rows was only half cleared)
    ws = og.Workspace()
    meth = {"full": og.OPH_METHOD_FULL, "goph": og.OPH_METHOD_GOPH, "hoph": og.OPH_METHOD_HOPH}[method]
    ws.get(og.oph_workspace_size_for(meth, q, s, prm, 0)).fill_(0xFF)
    fn(q, s, lay, prm, res, ws=ws)
    hist = res.hist().astype(np.int64)
    assert (hist == np.bincount(want["groups"].ravel(), minlength=len(hist))).all()
    n = res.n()
    out = og.Results(max(n, 1))
    og.topk_or_threshold_results(res, n, og.OPH_SELECT_THRESHOLD, out)
    got = out.numpy(n)
    assert list(zip(got["query"].tolist(), got["set_id"].tolist())) == oracle.threshold_list(want)
    assert n > 0
    sel = want[got["query"].astype(np.int64), got["set_id"].astype(np.int64)]
    for f in ("n_mb", "n_excl", "groups", "verdict", "flags"):
        assert (got[f].astype(np.int64) == sel[f].astype(np.int64)).all(), f
    assert np.abs(got["estimate"][sel["flags"] == 0] - sel["estimate"][sel["flags"] == 0]).max(initial=0) <= 1e-6
    brute = gpu_threshold_hits(method, q, s, layout=lay, strategy=og.OPH_STRATEGY_BRUTE, capacity=1 << 22, **kw)
    assert brute.tobytes() == got.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("lb,pipe", [("1", "1"), ("2", "1"), ("4", "1"), ("16", "1"), ("6", "0")])
def test_bitmap_goph_level_split(image_small, monkeypatch, lb, pipe):
    """GOPH through bit_pipe_kernel with the bitmap part forced to levels 1..lb (OPHGPU_GOPH_LB;
    lb = 1 and 2 are raised to the kernel's minimum of 64 bins) and every pair still undecided
    walked one by one over the later levels: dense records and threshold lists (with the
    termination histogram) == the oracle; pipe = 0 is the per-set bit_scan_q_kernel."""
    monkeypatch.setenv("OPHGPU_GOPH_LB", lb)
    monkeypatch.setenv("OPHGPU_BIT_PIPE", pipe)
    r, o, p = image_small, image_small["orc"], image_small["p"]
    lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
    for joint in (False, True):
        kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"], joint=joint, strategy=og.OPH_STRATEGY_BITMAP)
        n = 1000
        g = gpu_dense("goph", r["qo"], subview(r["so"], n), layout=lay, **kw)
        want = oracle_records("goph", o["QF"], o["F"][:n], k=p["k"], kprime=p["kprime"], **kw)
        assert_records_equal(g, want, f"goph lb={lb} joint={joint}")
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
    want = oracle_records("goph", o["QF"], o["F"], k=p["k"], kprime=p["kprime"], **kw)
    res = og.Results(1 << 22, stop_hist=True)
    og.compare_goph(r["qo"], r["so"], lay, og.params(p["t_num"], p["t_den"], p["eps"],
                                                     strategy=og.OPH_STRATEGY_BITMAP), res)
    hist = res.hist().astype(np.int64)
    assert (hist == np.bincount(want["groups"].ravel(), minlength=len(hist))).all()
    n = res.n()
    out = og.Results(max(n, 1))
    og.topk_or_threshold_results(res, n, og.OPH_SELECT_THRESHOLD, out)
    got = out.numpy(n)
    assert list(zip(got["query"].tolist(), got["set_id"].tolist())) == oracle.threshold_list(want)


def test_bitmap_domain_errors(tiny_run):
    """An explicit BITMAP request outside its domain fails (MinWise; |V| > 2^23); a
    workspace of only oph_workspace_size bytes is too small (OPH_ENOMEM) while AUTO
    then keeps the other strategies."""
    r, p = tiny_run, tiny_run["p"]
    prm = og.params(p["t_num"], p["t_den"], p["eps"], strategy=og.OPH_STRATEGY_BITMAP)
    with pytest.raises(og.OphError) as e:
        og.compare_minwise(r["qmw"], r["mw"], prm, og.Results(1 << 16))
    assert e.value.status == og.OPH_EINVAL
    lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
    class FixedWs(og.Workspace):  # a caller-owned workspace that does not grow
        def get(self, nbytes):
            return self.buf

    small = FixedWs()
    og.Workspace.get(small, og.oph_workspace_size(og.OPH_METHOD_FULL, r["qo"].n_sets, r["so"].n_sets, p["k"]))
    with pytest.raises(og.OphError) as e:
        og.compare_full(r["qo"], r["so"], lay, prm, og.Results(1 << 16), ws=small)
    assert e.value.status == og.OPH_ENOMEM
    og.compare_full(r["qo"], r["so"], lay, og.params(p["t_num"], p["t_den"], p["eps"]), og.Results(1 << 16), ws=small)
    V = 1 << 32
    offs, ids = make_csr([[1, 2, 3], [5, 6]])
    _, so, _ = gpu_build(offs, ids, V, 1, k=64, kprime=16)
    with pytest.raises(og.OphError) as e:
        og.compare_full(so, so, og.flat_layout(V, 64, 16), prm, og.Results(16))
    assert e.value.status == og.OPH_EINVAL


def test_validate_sets(monkeypatch):
    """oph_validate_sets (the CSR contract): valid collections pass; a repeated id,
    a decreasing pair and an id >= |V| are each reported (OPH_EINVAL); with OPHGPU_VALIDATE
    set the builds refuse such input."""
    V = 1000
    good_o, good_i = make_csr([[1, 2, 3], [], [999], [5, 7]])
    og.oph_validate_sets(og.SetCollection.from_numpy(good_o, good_i), V)
    bad = [np.array([1, 2, 2, 5], np.uint32), np.array([1, 3, 2, 5], np.uint32), np.array([1, 2, 3, 1000], np.uint32)]
    offs = np.array([0, 4], dtype=np.uint64)
    for ids in bad:
        with pytest.raises(og.OphError) as e:
            og.oph_validate_sets(og.SetCollection.from_numpy(offs, ids), V)
        assert e.value.status == og.OPH_EINVAL
    monkeypatch.setenv("OPHGPU_VALIDATE", "1")
    # (the environment variable is read once per process: a fresh interpreter)
    import subprocess
    import sys
    code = ("import numpy as np, paper_1805_11254_b200 as og; "
            "s = og.SetCollection.from_numpy(np.array([0, 3], np.uint64), np.array([4, 4, 9], np.uint32)); "
            "fl = og.flat_layout(1000, 8, 8)\n"
            "try:\n    og.oph_build_sketches(s, 1000, 1, flat=fl)\n    print('built')\n"
            "except og.OphError as e:\n    print('refused', e.status)\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert r.stdout.strip() == f"refused {og.OPH_EINVAL}", r.stdout + r.stderr


# ----------------------------------------------------------------------------- empty-aware HOPH (EH1-EH5)
@pytest.mark.parametrize("joint", [False, True])
def test_tiny_hoph_empty_aware(tiny_run, joint):
    """The empty-aware HOPH rule (OPH_VARIANT_EMPTY_AWARE on compare_hoph): dense records (every
    pair walked), termination histogram, and threshold lists through the join (pairs with a
    matched bin) and through the all-pairs walk (BRUTE) == the oracle's (O10e)."""
    r, o, p = tiny_run, tiny_run["orc"], tiny_run["p"]
    kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"], joint=joint)
    want = oracle_records("hoph_e", o["QH"], o["H"], kprime=p["hoph_kprime"], L=o["L"], **kw)
    g = gpu_dense("hoph_e", r["qh"], r["sh"], layout=r["hier"], **kw)
    assert_records_equal(g, want, f"tiny hoph_e joint={joint}")
    res = og.Results(1 << 20, stop_hist=True)
    og.compare_hoph(r["qh"], r["sh"], r["hier"], og.params(p["t_num"], p["t_den"], p["eps"], joint,
                                                           variant=og.OPH_VARIANT_EMPTY_AWARE), res)
    assert (res.hist().astype(np.int64) == np.bincount(want["groups"].ravel(), minlength=og.OPH_STOP_HIST_LEN)).all()
    for st in (og.OPH_STRATEGY_AUTO, og.OPH_STRATEGY_PROBE, og.OPH_STRATEGY_BRUTE):
        hits = gpu_threshold_hits("hoph_e", r["qh"], r["sh"], layout=r["hier"], strategy=st, **kw)
        assert [(int(h["query"]), int(h["set_id"])) for h in hits] == oracle.threshold_list(want), st
    # the variant differs from Algorithm 2 on these sparse sketches (it is not a no-op)
    paper = oracle_records("hoph", o["QH"], o["H"], kprime=p["hoph_kprime"], L=o["L"], **kw)
    assert (paper["groups"] != want["groups"]).any()


@pytest.mark.parametrize("V,hkp,seed", [(1000003, 8, 3), (4097, 32, 4), (1 << 20, 32, 5), (1 << 32, 32, 7)])
def test_hoph_empty_aware_ragged(V, hkp, seed):
    """Empty-aware HOPH dense records on ragged collections (empty sets / queries, non-power-of-
    two universes, 2^32), both empty modes."""
    rng = np.random.default_rng(seed + 100)
    sets = [rng.choice(V, size=int(s), replace=False) if s else [] for s in rng.integers(0, 60, size=300)]
    qsets = [sets[i] if i % 3 == 0 else rng.choice(V, size=int(rng.integers(0, 60)), replace=False)
             for i in range(37)]
    qsets[1] = []
    offs, ids = make_csr(sets)
    qoffs, qids = make_csr(qsets)
    hier = og.oph_hier_layout_make(V, 1, 1, hkp)
    _, _, sh = gpu_build(offs, ids, V, seed, hier=hier)
    _, _, qh = gpu_build(qoffs, qids, V, seed, hier=hier)
    glay = oracle.hoph_layout(V, 1, 1, hkp)
    H = oracle.hoph_sketch(offs, ids, V, glay, hkp, seed)
    QH = oracle.hoph_sketch(qoffs, qids, V, glay, hkp, seed)
    for joint in (False, True):
        kw = dict(t_num=7, t_den=10, eps=1e-4, joint=joint)
        assert_records_equal(gpu_dense("hoph_e", qh, sh, layout=hier, **kw),
                             oracle_records("hoph_e", QH, H, kprime=hkp, L=len(glay), **kw), f"hoph_e {V}")


# ----------------------------------------------------------------------------- build kernel variants (r02)
@pytest.mark.parametrize("V,k,hkp", [(1 << 16, 64, 16), (1 << 20, 512, 32), (1 << 32, 256, 32), (1 << 20, 512, 8),
                                     (1 << 20, 1024, 8), (1 << 12, 64, 2), (1 << 24, 32, 32), (1 << 16, 256, 4),
                                     (1 << 22, 2048, 8)])
@pytest.mark.parametrize("variant", ["default", "derive", "v1", "sb16_256", "sb8_256_derive"])
def test_build_variants_bit_exact(V, k, hkp, variant, monkeypatch):
    """Every build kernel of the power-of-two layout (warp-per-set, the same with the
    leading HOPH groups derived from the OPH minima (OPHGPU_BUILD_DERIVE), the r01
    element-strided kernel; tiles of 8 / 16 sets, 128 / 256 threads) gives the
    oracle's OPH and HOPH sketches.  Layouts span M_0 = k / 2k' OPH bins per derived
    HOPH bin of 2 .. 128 (lanes of 4 OPH bins: 1 .. 32 lanes per HOPH bin), k' < 4 (derivation
    off) and no derivable group at all."""
    env = dict(derive={"OPHGPU_BUILD_DERIVE": "1"}, v1={"OPHGPU_BUILD_V1": "1"},
               sb16_256={"OPHGPU_BUILD_SB": "16", "OPHGPU_BUILD_THREADS": "256"},
               sb8_256_derive={"OPHGPU_BUILD_THREADS": "256", "OPHGPU_BUILD_DERIVE": "1"}).get(variant, {})
    for kk, vv in env.items():
        monkeypatch.setenv(kk, vv)
    rng = np.random.default_rng(V % 1000 + k + hkp)
    nset = 1037  # not a multiple of 8 / 16 sets per tile
    sizes = rng.integers(0, 900, size=nset)
    sizes[[0, 5, 6, 7, 8, 100]] = 0  # empty sets inside a warp's pair, a whole empty tile row
    sizes[9] = 5000
    sets = [np.sort(rng.choice(V, size=min(int(s), V), replace=False)) if s else [] for s in sizes]
    offs, ids = make_csr(sets)
    hier = og.oph_hier_layout_make(V, 1, 1, hkp)
    _, so, sh = gpu_build(offs, ids, V, 11, k=k, kprime=8, hier=hier)
    F = oracle.oph_sketch(offs, ids, V, k, 11)
    glay = oracle.hoph_layout(V, 1, 1, hkp)
    H = oracle.hoph_sketch(offs, ids, V, glay, hkp, 11)
    assert (so.numpy() == F).all()
    assert (so.empty_numpy() == masks_from_values(F)).all()
    assert (sh.numpy() == H).all()
    assert (sh.empty_numpy() == masks_from_values(H)).all()


@pytest.mark.parametrize("joint", [False, True])
def test_full_oph_exit_exact(image_small, monkeypatch, joint):
    """R32: full OPH's BITMAP scan stops a set once no pair of the query block can reach T
    (count + the set's non-empty bins left < a lower bound of every threshold).  The threshold
    list and the histogram are byte-identical to the scan of every bin (OPHGPU_FULL_EXIT=0)
    and to the oracle; d_bins_scanned counts the rows gathered: every (set, bin) of both
    query blocks without the exit, fewer with it."""
    r, o, p = image_small, image_small["orc"], image_small["p"]
    q, s = r["qo"], r["so"]
    lay = og.flat_layout(r["w"].vocab_size, p["k"], p["kprime"])
    prm = og.params(p["t_num"], p["t_den"], p["eps"], joint, og.OPH_STRATEGY_BITMAP)
    runs = {}
    for env in ("1", "0", "from64", "from32"):
        monkeypatch.setenv("OPHGPU_FULL_EXIT", "0" if env == "0" else "1")
        if env.startswith("from"):  # R32b's prefix bounds checked at every 32 bins (from 64: the
            # next set's lookups are fetched ahead at bin 32; from 32: no room for that, none fetched)
            monkeypatch.setenv("OPHGPU_FULL_EXIT_FROM", env[4:])
        res = og.Results(1 << 22, stop_hist=True, bins_scanned=True)
        og.compare_full(q, s, lay, prm, res)
        n = res.n()
        out = og.Results(max(n, 1))
        og.topk_or_threshold_results(res, n, og.OPH_SELECT_THRESHOLD, out)
        runs[env] = (out.numpy(n).tobytes(), res.hist().tobytes(), int(res.bins_scanned.item()), n)
    want = oracle_records("full", o["QF"], o["F"], k=p["k"], kprime=p["kprime"], t_num=p["t_num"],
                          t_den=p["t_den"], eps=p["eps"], joint=joint)
    assert runs["1"][0] == runs["0"][0] and runs["1"][1] == runs["0"][1]
    assert runs["from32"][0] == runs["0"][0] and runs["from32"][1] == runs["0"][1]
    assert runs["from64"][0] == runs["0"][0] and runs["from64"][1] == runs["0"][1]
    assert runs["from32"][2] <= runs["1"][2]
    assert runs["1"][3] == len(oracle.threshold_list(want)) > 0
    blocks = -(-q.n_sets // 2048)
    assert runs["0"][2] == s.n_sets * p["k"] * blocks
    assert 0 < runs["1"][2] < runs["0"][2]


@pytest.mark.parametrize("exit_from", [None, "32", "64"])
@pytest.mark.parametrize("tn,td", [(7, 10), (1, 20), (9, 10), (1, 1)])
@pytest.mark.parametrize("joint", [False, True])
def test_full_oph_exit_ragged(tn, td, joint, exit_from, monkeypatch):
    """R32 / R32b on a ragged collection (517 sets: not a whole number of 8-set tiles; empty
    sets, a whole-universe-sized set, 45 queries incl. exact copies and an empty query) at
    k = 512, thresholds from 1/20 (almost no set exits) to 1 (almost every set exits at the
    first check), the exit checked from bin 288 (default: ceil32(9 k / 16)) or at every 32 bins from bin 32
    (the prefix bounds R32b at every checkpoint): the BITMAP threshold list == BRUTE's ==
    the oracle's."""
    if exit_from:
        monkeypatch.setenv("OPHGPU_FULL_EXIT_FROM", exit_from)
    rng = np.random.default_rng(tn * 100 + td + joint)
    V, k, kp = 1 << 20, 512, 32
    sizes = rng.integers(0, 700, size=517)
    sizes[:3] = 0
    sizes[7] = 20000
    sets = [rng.choice(V, size=int(s), replace=False) if s else [] for s in sizes]
    qsets = [sets[i] if i % 3 == 0 else rng.choice(V, size=int(rng.integers(0, 700)), replace=False)
             for i in range(45)]
    qsets[1] = []
    offs, ids = make_csr(sets)
    qoffs, qids = make_csr(qsets)
    _, so, _ = gpu_build(offs, ids, V, 5, k=k, kprime=kp)
    _, qo, _ = gpu_build(qoffs, qids, V, 5, k=k, kprime=kp)
    lay = og.flat_layout(V, k, kp)
    kw = dict(t_num=tn, t_den=td, joint=joint)
    bit = gpu_threshold_hits("full", qo, so, layout=lay, strategy=og.OPH_STRATEGY_BITMAP, **kw)
    brute = gpu_threshold_hits("full", qo, so, layout=lay, strategy=og.OPH_STRATEGY_BRUTE, **kw)
    assert bit.tobytes() == brute.tobytes()
    want = oracle_records("full", oracle.oph_sketch(qoffs, qids, V, k, 5), oracle.oph_sketch(offs, ids, V, k, 5),
                          k=k, kprime=kp, **kw)
    assert [(int(h["query"]), int(h["set_id"])) for h in bit] == oracle.threshold_list(want)
