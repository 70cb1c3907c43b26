"""A/B sweep of the OPH+HOPH build tile (sets per CTA x threads) on image-like and text-like."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1805_11254_b200 as og
from workloads import gen_gpu, text_like

out = {}
for name, w in (("image-like", gen_gpu.image_like()), ("text-like", text_like())):
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    flat = og.flat_layout(V, p["k"], p["kprime"])
    hier = og.oph_hier_layout_make(V, 1, 1, p["hoph_kprime"])
    sets = og.SetCollection.from_numpy(w.offsets, w.ids)
    so, sh = og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier)
    ref = (so.values.clone(), sh.values.clone())
    for sb in (4, 8, 16):
        for th in (128, 256, 512):
            os.environ["OPHGPU_BUILD_SB"], os.environ["OPHGPU_BUILD_THREADS"] = str(sb), str(th)
            ts = []
            for _ in range(6):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier, out_oph=so, out_hoph=sh)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ok = bool((so.values == ref[0]).all()) and bool((sh.values == ref[1]).all())
            out[f"{name} SB={sb} T={th}"] = (min(ts[1:]), ok)
            print(name, sb, th, round(min(ts[1:]), 4), ok, flush=True)
json.dump(out, open("gpurun_out/build_sweep.json", "w"), indent=1)
