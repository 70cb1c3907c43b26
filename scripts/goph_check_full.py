"""GOPH on the full sweep-0.9 bench configuration (2M sets x 256 queries, survivor capacity
2^28): hit lists of sampled queries vs the oracle, for the current BRUTE path."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1805_11254_b200 as og  # noqa: E402
from workloads.gen_gpu import sweep  # noqa: E402

w = sweep(0.9, n_sets=2_000_000, n_queries=256)
p = w.params
V, seed = w.vocab_size, p["perm_seed"]
flat = og.flat_layout(V, p["k"], p["kprime"])
sets = og.SetCollection.from_numpy(w.offsets, w.ids)
qs = og.SetCollection.from_numpy(w.q_offsets, w.q_ids)
so, _ = og.oph_build_sketches(sets, V, seed, flat=flat)
qo, _ = og.oph_build_sketches(qs, V, seed, flat=flat)
prm = og.params(p["t_num"], p["t_den"], p["eps"], strategy=og.OPH_STRATEGY_BRUTE)
res = og.Results(1 << 25)
og.compare_goph(qo, so, flat, prm, res, survivor_capacity=1 << 28)
n = res.n()
h = res.numpy(min(n, 1 << 25))
tag = "old" if os.environ.get("OPHGPU_NO_MULTI_LEVEL_SCAN") else "multi"
print(f"{tag}: total hits {n}")
sample = [0, 1, 100, 128, 200, 255]
F = oracle.oph_sketch(w.offsets, w.ids, V, p["k"], seed)
QF = oracle.oph_sketch(w.q_offsets, w.q_ids, V, p["k"], seed)
for q in sample:
    want = oracle.compare_goph(QF[q:q + 1], F, n=p["k"] // p["kprime"], kprime=p["kprime"], t_num=p["t_num"],
                               t_den=p["t_den"], eps=p["eps"])
    wl = [s for _, s in oracle.threshold_list(want, 0)]
    gl = sorted(h["set_id"][h["query"] == q].tolist())
    print(f"  q{q}: gpu {len(gl)} oracle {len(wl)} equal {gl == wl}")
