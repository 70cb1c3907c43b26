"""Query-block sweep of the BRUTE collection scan: full OPH on the
image-like collection (10^6 sets x 512 bins, 2.1 GB) for Q = 4 .. 256 queries.
Per Q: the scan kernel's device time (CUPTI), the collection bytes it streamed
(one pass per 32-query block, or one pass for Q <= 32 with B = Q), the effective
HBM GB/s and bin-compares/s."""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_11254_b200 as og  # noqa: E402
from workloads import gen_gpu  # noqa: E402

w = gen_gpu.image_like()
p = w.params
V, seed, k, kp = w.vocab_size, p["perm_seed"], p["k"], p["kprime"]
flat = og.flat_layout(V, k, kp)
sets = og.SetCollection.from_numpy(w.offsets, w.ids)
so, _ = og.oph_build_sketches(sets, V, seed, flat=flat)
N = so.n_sets
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
hbm = peaks["hbm_gbs"]
qs_all = og.SetCollection.from_numpy(w.q_offsets, w.q_ids)
qo_all, _ = og.oph_build_sketches(qs_all, V, seed, flat=flat)
prm = og.params(p["t_num"], p["t_den"], p["eps"], strategy=og.OPH_STRATEGY_BRUTE)
res = og.Results(1 << 24)
ws = og.Workspace()
only = [int(x) for x in sys.argv[1:]] or [4, 8, 16, 32, 64, 128, 256]
for Q in only:
    q = og.Sketches(qo_all.values, qo_all.empty, None, Q, k, seed, V)
    for _ in range(2):
        res.reset()
        og.compare_full(q, so, flat, prm, res, ws=ws)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        res.reset()
        og.compare_full(q, so, flat, prm, res, ws=ws)
        torch.cuda.synchronize()
    us = sum(e.device_time_total for e in prof.events() if "scan_kernel" in e.name)
    B = 32 if Q > 16 else max(4, 1 << (Q - 1).bit_length())
    passes = -(-Q // B)
    by = passes * N * (4 * k + 4 * (k // 32))
    print(json.dumps({"Q": Q, "B": B, "scan_us": round(us, 1), "passes": passes,
                      "GBps": round(by / us / 1e3, 1), "hbm_frac": round(by / us / 1e3 / hbm, 3),
                      "bin_compares_per_s": Q * N * k / (us / 1e6)}))
