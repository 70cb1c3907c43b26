"""A/B of the OPH+HOPH build kernels on image-like, text-like and a scale shard:
r01 element-strided kernel (OPHGPU_BUILD_V1) vs the r02 warp-per-set kernel with and
without the derived HOPH groups, tiles of 8 / 16 sets x 128 / 256 threads.  Every
variant's sketches must equal the r01 kernel's (the parity suite ties that to the oracle)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1805_11254_b200 as og
from workloads import gen_gpu, text_like

VARIANTS = {
    "v1 SB8 T128": {"OPHGPU_BUILD_V1": "1"},
    "warp SB8 T128": {},
    "warp SB8 T128 derive": {"OPHGPU_BUILD_DERIVE": "1"},
    "warp SB8 T256": {"OPHGPU_BUILD_THREADS": "256"},
    "warp SB16 T256": {"OPHGPU_BUILD_SB": "16", "OPHGPU_BUILD_THREADS": "256"},
    "warp SB16 T128": {"OPHGPU_BUILD_SB": "16", "OPHGPU_BUILD_THREADS": "128"},
}
KEYS = ("OPHGPU_BUILD_V1", "OPHGPU_BUILD_DERIVE", "OPHGPU_BUILD_SB", "OPHGPU_BUILD_THREADS")
out = {}
cfgs = (("image-like", gen_gpu.image_like), ("text-like", text_like), ("scale-shard", gen_gpu.scale_shard))
for name, mk in cfgs:
    w = mk()
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    flat = og.flat_layout(V, p["k"], p["kprime"])
    hier = og.oph_hier_layout_make(V, 1, 1, p["hoph_kprime"])
    sets = og.SetCollection.from_numpy(w.offsets, w.ids) if not torch.is_tensor(w.offsets) else \
        og.SetCollection(w.offsets, w.ids)
    ref = None
    n = sets.n_sets
    nbytes = int(sets.ids.numel()) * 4 + (int(sets.offsets.numel())) * 8
    for vname, env in VARIANTS.items():
        for kk in KEYS:
            os.environ.pop(kk, None)
        os.environ.update(env)
        so, sh = og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier)
        torch.cuda.synchronize()
        if ref is None:
            ref = tuple(x[:, :n].clone() for x in (so.values, sh.values, so.empty, sh.empty))
        # (columns past n_sets are padding of ld, never written)
        ok = all(bool((x[:, :n] == y).all()) for x, y in zip((so.values, sh.values, so.empty, sh.empty), ref))
        ts = []
        for _ in range(8):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier, out_oph=so, out_hoph=sh)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ob = so.values.numel() * 4 + sh.values.numel() * 4 + so.empty.numel() * 4 + sh.empty.numel() * 4
        t = sorted(ts[1:])[len(ts[1:]) // 2]
        out[f"{name} | {vname}"] = dict(ms=t, ok=ok, gbps=(nbytes + ob) / t / 1e6)
        print(name, "|", vname, round(t, 4), "ms", round((nbytes + ob) / t / 1e6, 1), "GB/s", ok, flush=True)
    del sets, so, sh, ref, w
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/build_ab.json", "w"), indent=1)
