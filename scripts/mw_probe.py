"""Time minwise_build_sketches on the text-like (|V| = 2^32) or image-like (|V| = 2^20)
collection with CUDA events; prints a checksum so build variants can be compared."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_11254_b200 as og  # noqa: E402
from workloads import gen_gpu, text_like  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "text"
w = text_like() if cfg == "text" else gen_gpu.image_like()
p = w.params
V, seed = w.vocab_size, p["perm_seed"]
sets = og.SetCollection.from_numpy(w.offsets, w.ids)
mw = og.minwise_build_sketches(sets, V, seed, p["mw_k"])
times = []
for rep in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    og.minwise_build_sketches(sets, V, seed, p["mw_k"], out=mw)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
print(f"{cfg} minwise build: {sorted(times)[1]:.3f} ms, checksum {int(mw.values.to(torch.int64).sum())}")
