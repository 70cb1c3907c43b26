"""Time one compare_* call (CUDA events, median of reps) on the text-like or image-like
workload and list its kernels with CUPTI device times (A/B of path changes)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_11254_b200 as og  # noqa: E402
from workloads import gen_gpu, text_like  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="image")
ap.add_argument("--methods", default="goph,hoph")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--strategy", type=int, default=og.OPH_STRATEGY_AUTO)
ap.add_argument("--variant", type=int, default=0, help="1: the empty-aware GOPH rule")
ap.add_argument("--queries", type=int, default=0, help="sweep configs: the number of queries (default 1,024)")
args = ap.parse_args()
if args.config == "text":
    w = text_like()
elif args.config == "scale":
    w = gen_gpu.scale_shard()
elif args.config.startswith("sweep"):
    w = gen_gpu.sweep(float(args.config[5:]), **({"n_queries": args.queries} if args.queries else {}))
else:
    w = gen_gpu.image_like()
p = w.params
V, seed = w.vocab_size, p["perm_seed"]
hier = og.oph_hier_layout_make(V, 1, 1, p["hoph_kprime"])
flat = og.flat_layout(V, p["k"], p["kprime"])
sets = og.SetCollection.from_numpy(w.offsets, w.ids)
qs = og.SetCollection.from_numpy(w.q_offsets, w.q_ids)
so, sh = og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier)
qo, qh = og.oph_build_sketches(qs, V, seed, flat=flat, hier=hier)
prm = og.params(p["t_num"], p["t_den"], p["eps"], strategy=args.strategy)
prm_e = og.params(p["t_num"], p["t_den"], p["eps"], strategy=args.strategy, variant=args.variant)
res = og.Results(1 << 24)
ws = og.Workspace()
cap = min(((qo.n_sets + 31) // 32) * 32 * so.n_sets, 1 << 26)
for m in args.methods.split(","):
    fn = {"full": lambda: og.compare_full(qo, so, flat, prm, res, ws=ws),
          "goph": lambda: og.compare_goph(qo, so, flat, prm_e, res, ws=ws, survivor_capacity=cap),
          "hoph": lambda: og.compare_hoph(qh, sh, hier, prm, res, ws=ws, survivor_capacity=cap)}[m]
    ts = []
    for r in range(args.reps):
        res.reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{args.config} {m}: {sorted(ts)[len(ts) // 2]:.3f} ms, hits {res.n()}")
    from torch.profiler import ProfilerActivity, profile
    res.reset()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    agg = {}
    for ev in prof.events():
        if ev.device_type.name == "CUDA":
            k = ev.name.split("(")[0][-40:]
            c = agg.setdefault(k, [0, 0.0])
            c[0] += 1
            c[1] += ev.device_time_total
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:5]:
        print(f"   {k:40s} n={n:3d} {t:10.1f} us")
