"""Throughput of shingle_text on ~200 MB of synthetic text (CUDA events)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_11254_b200 as og  # noqa: E402

rng = np.random.default_rng(0)
vocab = np.array([("w%d" % i).encode() for i in range(50_000)], dtype=object)
n_docs, words_per_doc = 200_000, 160
lens = np.array([len(v) for v in vocab])
idx = rng.integers(0, len(vocab), size=n_docs * words_per_doc)
# bytes: words separated by single spaces, documents concatenated
word_bytes = np.frombuffer(b"".join(vocab[idx] + b" "), dtype=np.uint8)
doc_len = np.add.reduceat(lens[idx] + 1, np.arange(0, len(idx), words_per_doc))
offs = np.zeros(n_docs + 1, dtype=np.int64)
np.cumsum(doc_len, out=offs[1:])
text = torch.from_numpy(word_bytes.copy()).cuda()
o = torch.from_numpy(offs).cuda()
ws = og.Workspace()
for w in (1, 3, 5):
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sets = og.shingle_text(text, o, w, 1 << 32, 7, ws=ws)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"w={w}: {text.numel() / 1e6:.0f} MB, {n_docs} docs, {sets.ids.numel()} ids: {ms:.2f} ms "
          f"= {text.numel() / ms / 1e6:.1f} GB/s of text, {n_docs / ms * 1e3:.3e} docs/s")
