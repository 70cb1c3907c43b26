"""Time oph_build_sketches (OPH + HOPH) on the text-like collection (CUDA events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_11254_b200 as og  # noqa: E402
from workloads import text_like  # noqa: E402

w = text_like()
p = w.params
V, seed = w.vocab_size, p["perm_seed"]
hier = og.oph_hier_layout_make(V, 1, 1, p["kprime"])
flat = og.flat_layout(V, p["k"], p["kprime"])
sets = og.SetCollection.from_numpy(w.offsets, w.ids)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    so, sh = og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier)
    e1.record()
    torch.cuda.synchronize()
    print(f"build rep {rep}: {e0.elapsed_time(e1):.3f} ms, checksum {int(so.values.to(torch.int64).sum()) ^ int(sh.values.to(torch.int64).sum())}")
