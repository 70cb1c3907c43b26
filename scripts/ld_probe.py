"""Does the build slow down with the sketch matrices' row stride (ld) alone?  The text-like
collection (200,000 sets) built into matrices of ld = 200,000 and ld = 1,250,016 (the scale
shard's): same work, rows 0.8 MB vs 5 MB apart (one 2-MB page per row per CTA write-out)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1805_11254_b200 as og
from paper_1805_11254_b200 import lib, oph_perm, OPH_PERM_KEYED, _ptr, c_u64, _check
from workloads import text_like

w = text_like()
p = w.params
V, seed = w.vocab_size, p["perm_seed"]
flat = og.flat_layout(V, p["k"], p["kprime"])
hier = og.oph_hier_layout_make(V, 1, 1, p["hoph_kprime"])
sets = og.SetCollection.from_numpy(w.offsets, w.ids)
perm = oph_perm(V, seed, OPH_PERM_KEYED, 0)
nbh = hier.L * hier.kprime
for ld in (sets.n_sets, 1_250_016, 4_000_000):
    ld = (ld + 31) // 32 * 32
    ov = torch.empty((p["k"], ld), dtype=torch.int32, device="cuda")
    oe = torch.empty(((p["k"] + 31) // 32, ld), dtype=torch.int32, device="cuda")
    hv = torch.empty((nbh, ld), dtype=torch.int32, device="cuda")
    he = torch.empty(((nbh + 31) // 32, ld), dtype=torch.int32, device="cuda")
    ts = []
    for r in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _check(lib().oph_build_sketches(ctypes.byref(sets.c()), ctypes.byref(perm), ctypes.byref(flat), _ptr(ov),
                                        _ptr(oe), ctypes.byref(hier), _ptr(hv), _ptr(he), c_u64(ld), None), "build")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"ld {ld}: {sorted(ts[1:])[3]:.4f} ms", flush=True)
    del ov, oe, hv, he
    torch.cuda.empty_cache()
