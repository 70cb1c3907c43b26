"""Debug: BITMAP full-OPH threshold list vs dense records vs the oracle on an image-like sample."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle
import paper_1805_11254_b200 as og
from workloads import gen
from gpu_helpers import gpu_build, oracle_records, gpu_dense

w = gen.image_like(n_sets=20_000, n_queries=2100)
p = w.params
V, seed = w.vocab_size, p["perm_seed"]
_, so, _ = gpu_build(w.offsets, w.ids, V, seed, k=p["k"], kprime=p["kprime"])
_, qo, _ = gpu_build(w.q_offsets, w.q_ids, V, seed, k=p["k"], kprime=p["kprime"])
lay = og.flat_layout(V, p["k"], p["kprime"])
kw = dict(t_num=p["t_num"], t_den=p["t_den"], eps=p["eps"])
F = oracle.oph_sketch(w.offsets, w.ids, V, p["k"], seed)
QF = oracle.oph_sketch(w.q_offsets, w.q_ids, V, p["k"], seed)
want = oracle_records("full", QF, F, k=p["k"], kprime=p["kprime"], **kw)
res = og.Results(1 << 22)
og.compare_full(qo, so, lay, og.params(p["t_num"], p["t_den"], p["eps"], strategy=og.OPH_STRATEGY_BITMAP), res)
n = res.n()
h = res.numpy(n)
print("gpu hits", n, "oracle hits", int(want["verdict"].sum()))
bad = [(int(a), int(b)) for a, b in zip(h["query"], h["set_id"]) if want["verdict"][a, b] != 1]
print("bad", len(bad), bad[:10])
for a, b in bad[:5]:
    r = h[(h["query"] == a) & (h["set_id"] == b)][0]
    print("gpu", r, "oracle", want[a, b])
from collections import Counter
print("bad queries", Counter(a for a, b in bad).most_common(10))
print("bad query words", Counter((a % 2048) // 32 for a, b in bad).most_common(10))
d = gpu_dense("full", qo, so, layout=lay, strategy=og.OPH_STRATEGY_BITMAP, **kw)
diff = np.nonzero(d["n_mb"].astype(np.int64) != want["n_mb"].astype(np.int64))
print("dense n_mb diffs", len(diff[0]), list(zip(diff[0][:10].tolist(), diff[1][:10].tolist())))
