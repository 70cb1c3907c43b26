"""A/B check of the GOPH BRUTE paths (multi-level scan vs scan + survivor levels) against
the oracle on a reduced sweep-0.9 instance with several query chunks."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1805_11254_b200 as og  # noqa: E402
from workloads.gen_gpu import sweep  # noqa: E402

method = sys.argv[1] if len(sys.argv) > 1 else "goph"
w = sweep(0.9, n_sets=60_000, n_queries=256)
p = w.params
V, seed = w.vocab_size, p["perm_seed"]
flat = og.flat_layout(V, p["k"], p["kprime"])
hier = og.oph_hier_layout_make(V, 1, 1, p["kprime"])
sets = og.SetCollection.from_numpy(w.offsets, w.ids)
qs = og.SetCollection.from_numpy(w.q_offsets, w.q_ids)
so, sh = og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier)
qo, qh = og.oph_build_sketches(qs, V, seed, flat=flat, hier=hier)
prm = og.params(p["t_num"], p["t_den"], p["eps"], strategy=og.OPH_STRATEGY_BRUTE)
res = og.Results(1 << 24)
if method == "goph":
    og.compare_goph(qo, so, flat, prm, res, survivor_capacity=60_000 * 64)
else:
    og.compare_hoph(qh, sh, hier, prm, res, survivor_capacity=60_000 * 64)
n = res.n()
h = res.numpy(n)
got = sorted(zip(h["query"].tolist(), h["set_id"].tolist()))
if method == "goph":
    F = oracle.oph_sketch(w.offsets, w.ids, V, p["k"], seed)
    QF = oracle.oph_sketch(w.q_offsets, w.q_ids, V, p["k"], seed)
    want = oracle.compare_goph(QF, F, n=p["k"] // p["kprime"], kprime=p["kprime"], t_num=p["t_num"], t_den=p["t_den"],
                               eps=p["eps"])
else:
    lay = oracle.hoph_layout(V, 1, 1, p["kprime"])
    H = oracle.hoph_sketch(w.offsets, w.ids, V, lay, p["kprime"], seed)
    QH = oracle.hoph_sketch(w.q_offsets, w.q_ids, V, lay, p["kprime"], seed)
    want = oracle.compare_hoph(QH, H, L=len(lay), kprime=p["kprime"], a=1, b=1, t_num=p["t_num"], t_den=p["t_den"],
                               eps=p["eps"])
wl = oracle.threshold_list(want, 0)
tag = "old" if os.environ.get("OPHGPU_NO_MULTI_LEVEL_SCAN") else "multi"
print(f"{method} {tag}: gpu hits {len(got)} oracle {len(wl)} equal {got == wl}")
if got != wl:
    g, o = set(got), set(wl)
    print("  only gpu:", len(g - o), sorted(g - o)[:5], " only oracle:", len(o - g), sorted(o - g)[:5])
