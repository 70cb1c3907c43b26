"""Build both layouts in one pass vs one pass per layout (OPH rows, then HOPH rows), at the
text-like collection's own ld (2e5) and at the scale shard's (1.25e6): does halving the rows
a pass writes pay for reading and hashing the ids twice?"""
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


def timeit(fn, reps=8):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts[1:])[len(ts[1:]) // 2]


for ld in (sets.n_sets, 1_250_016):
    ld = (ld + 31) // 32 * 32
    ov = torch.empty((p["k"], ld), dtype=torch.int32, device="cuda")
    oe = torch.empty(((p["k"] + 31) // 32, ld), dtype=torch.int32, device="cuda")
    hv = torch.empty((nbh, ld), dtype=torch.int32, device="cuda")
    he = torch.empty(((nbh + 31) // 32, ld), dtype=torch.int32, device="cuda")
    both = lambda: _check(lib().oph_build_sketches(ctypes.byref(sets.c()), ctypes.byref(perm), ctypes.byref(flat),
                                                   _ptr(ov), _ptr(oe), ctypes.byref(hier), _ptr(hv), _ptr(he),
                                                   c_u64(ld), None), "both")
    only_f = lambda: _check(lib().oph_build_sketches(ctypes.byref(sets.c()), ctypes.byref(perm), ctypes.byref(flat),
                                                     _ptr(ov), _ptr(oe), None, None, None, c_u64(ld), None), "flat")
    only_h = lambda: _check(lib().oph_build_sketches(ctypes.byref(sets.c()), ctypes.byref(perm), None, None, None,
                                                     ctypes.byref(hier), _ptr(hv), _ptr(he), c_u64(ld), None), "hier")
    tb = timeit(both)
    tf = timeit(only_f)
    th = timeit(only_h)
    print(f"ld {ld}: both {tb:.4f} ms | flat only {tf:.4f} + hier only {th:.4f} = {tf + th:.4f} ms", flush=True)
    del ov, oe, hv, he
    torch.cuda.empty_cache()
