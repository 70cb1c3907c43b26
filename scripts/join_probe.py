"""Time one compare_* call of the text-like workload (PROBE strategy) with CUDA
events; used for quick iterations and as the ncu target of the join kernel."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_11254_b200 as og  # noqa: E402
from workloads import text_like  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--method", default="full")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--strategy", type=int, default=og.OPH_STRATEGY_PROBE)
args = ap.parse_args()

w = text_like()
p = w.params
V, seed = w.vocab_size, p["perm_seed"]
hier = og.oph_hier_layout_make(V, 1, 1, p["kprime"])
flat = og.flat_layout(V, p["k"], p["kprime"])
sets = og.SetCollection.from_numpy(w.offsets, w.ids)
qs = og.SetCollection.from_numpy(w.q_offsets, w.q_ids)
so, sh = og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier)
qo, qh = og.oph_build_sketches(qs, V, seed, flat=flat, hier=hier)
prm = og.params(p["t_num"], p["t_den"], p["eps"], strategy=args.strategy)
res = og.Results(1 << 22)
if args.method == "minwise":
    mw = og.minwise_build_sketches(sets, V, seed, p["mw_k"])
    qmw = og.minwise_build_sketches(qs, V, seed, p["mw_k"])
fn = {"minwise": lambda: og.compare_minwise(qmw, mw, prm, res),
      "full": lambda: og.compare_full(qo, so, flat, prm, res),
      "goph": lambda: og.compare_goph(qo, so, flat, prm, res),
      "hoph": lambda: og.compare_hoph(qh, sh, hier, prm, res)}[args.method]
torch.cuda.synchronize()
for r in range(args.reps):
    res.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{args.method} rep {r}: {e0.elapsed_time(e1):.3f} ms, hits {res.n()}")

# per-kernel device times of one more call (CUPTI via torch.profiler)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

res.reset()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    fn()
    torch.cuda.synchronize()
for ev in prof.events():
    if ev.device_type.name == "CUDA":
        print(f"  kernel {ev.name[:60]:60s} {ev.device_time_total:9.1f} us")
