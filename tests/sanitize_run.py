"""Small end-to-end run of every kernel for compute-sanitizer (not a pytest file):

    compute-sanitizer --tool memcheck python tests/sanitize_run.py

Tiny config: builds (OPH, HOPH, MinWise), every compare in dense and in
threshold mode with both scan strategies (PROBE incl. its BRUTE list fallback
and the survivor levels), threshold and top-k selection, the 4 / 8 / 16-query scan blocks, exact Jaccard
pairs and text shingling."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1805_11254_b200 as og  # noqa: E402
from workloads import tiny  # noqa: E402


def main():
    w = tiny()
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    hier = og.oph_hier_layout_make(V, 1, 1, p["hoph_kprime"])
    flat = og.flat_layout(V, p["k"], p["kprime"])
    sets = og.SetCollection.from_numpy(w.offsets, w.ids)
    # 40 copies of query 0 force PROBE overflow -> BRUTE list scan
    qo_np = [w.query_ids(q) for q in range(w.n_queries)] + [w.query_ids(0)] * 40
    qoff = np.zeros(len(qo_np) + 1, dtype=np.uint64)
    np.cumsum([len(x) for x in qo_np], out=qoff[1:])
    qs = og.SetCollection.from_numpy(qoff, np.concatenate(qo_np))
    so, sh = og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier)
    qo, qh = og.oph_build_sketches(qs, V, seed, flat=flat, hier=hier)
    mw = og.minwise_build_sketches(sets, V, seed, p["mw_k"])
    qmw = og.minwise_build_sketches(qs, V, seed, p["mw_k"])
    total = 0
    for strategy in (og.OPH_STRATEGY_BRUTE, og.OPH_STRATEGY_PROBE):
        prm = og.params(p["t_num"], p["t_den"], p["eps"], strategy=strategy)
        for dense in (False, True):
            for name, fn, args in [("full", og.compare_full, (qo, so, flat)), ("goph", og.compare_goph, (qo, so, flat)),
                                   ("hoph", og.compare_hoph, (qh, sh, hier))]:
                r = og.Results(qo.n_sets * so.n_sets if dense else 1 << 16, dense=dense)
                fn(*args, prm, r)
                total += r.n()
            r = og.Results(qo.n_sets * so.n_sets if dense else 1 << 16, dense=dense)
            og.compare_minwise(qmw, mw, prm, r)
            n = r.n()
            total += n
            if not dense:
                out = og.Results(max(n, 1))
                og.topk_or_threshold_results(r, n, og.OPH_SELECT_THRESHOLD, out)
                og.topk_or_threshold_results(r, n, og.OPH_SELECT_TOPK, out, topk=3, k_bins=p["mw_k"])
    # small query blocks of the BRUTE scan (4 / 8 / 16 queries per register block)
    import dataclasses
    prm = og.params(p["t_num"], p["t_den"], p["eps"], strategy=og.OPH_STRATEGY_BRUTE)
    for nq in (3, 8, 13):
        q = dataclasses.replace(qo, n_sets=nq)
        for fn in (og.compare_full, og.compare_goph):
            r = og.Results(nq * so.n_sets, dense=True)
            fn(q, so, flat, prm, r)
            total += r.n()
    # exact Jaccard of some pairs, and the text shingling front end
    qi = torch.arange(0, 64, dtype=torch.int32, device="cuda") % w.n_queries
    si = (torch.arange(0, 64, dtype=torch.int32, device="cuda") * 31) % w.n_sets
    inter, union = og.exact_jaccard_pairs(qs, sets, qi, si)
    total += int(inter.sum().item())
    docs = [b"the quick brown fox jumps over the lazy dog", b"", b"  a b  ", b"Lorem ipsum dolor sit amet, consectetur"]
    text = torch.tensor(list(b"".join(docs)), dtype=torch.uint8, device="cuda")
    offs = torch.tensor(np.cumsum([0] + [len(d) for d in docs]), dtype=torch.int64, device="cuda")
    sh_sets = og.shingle_text(text, offs, 3, 1 << 20, 7)
    total += int(sh_sets.n_sets)
    # BITMAP at image-like widths (k = 512, two 2,048-query blocks, the second ragged): the
    # pipelined full-OPH scan with its exact exit (R32) and GOPH / HOPH, plus the r02 build
    # kernel (warp per set) with and without the derived HOPH groups
    from workloads import gen
    wi = gen.image_like(n_sets=3000, n_queries=2100, planted_per_query=0)
    pi = wi.params
    Vi, si_ = wi.vocab_size, pi["perm_seed"]
    hier_i = og.oph_hier_layout_make(Vi, 1, 1, pi["hoph_kprime"])
    flat_i = og.flat_layout(Vi, pi["k"], pi["kprime"])
    sets_i = og.SetCollection.from_numpy(wi.offsets, wi.ids)
    qs_i = og.SetCollection.from_numpy(wi.q_offsets, wi.q_ids)
    for derive in ("0", "1"):
        os.environ["OPHGPU_BUILD_DERIVE"] = derive
        so_i, sh_i = og.oph_build_sketches(sets_i, Vi, si_, flat=flat_i, hier=hier_i)
    os.environ.pop("OPHGPU_BUILD_DERIVE", None)
    qo_i, qh_i = og.oph_build_sketches(qs_i, Vi, si_, flat=flat_i, hier=hier_i)
    prm_b = og.params(pi["t_num"], pi["t_den"], pi["eps"], strategy=og.OPH_STRATEGY_BITMAP)
    for fn, q_, s_, lay in ((og.compare_full, qo_i, so_i, flat_i), (og.compare_goph, qo_i, so_i, flat_i),
                            (og.compare_hoph, qh_i, sh_i, hier_i)):
        r = og.Results(1 << 20, stop_hist=True, bins_scanned=True)
        fn(q_, s_, lay, prm_b, r)
        total += r.n() + int(r.bins_scanned.item())
    torch.cuda.synchronize()
    print("sanitize_run ok", total)


if __name__ == "__main__":
    main()
