"""Oracle (test infrastructure only; see oracle/__init__.py): text shingling,
the ingestion step before the OPH build (SPEC shingle_text;
the paper's "convert the words of each document into a set of fingerprints",
P:53).  Plain Python, written from the definition in DESIGN.md section 4b:

  tokens  = maximal runs of non-whitespace bytes (ASCII whitespace: space, \\t,
            \\n, \\v, \\f, \\r), ASCII letters lowercased
  tok(t)  = FNV-1a 64 of the token's bytes
  gram    = w consecutive tokens of one document (a document with fewer than
            w tokens has none)
  h_0 = seed;  h_i = mix64(h_{i-1} + GOLDEN + tok(t_i)) for i = 1..w
  id      = h_w mod vocab_size
  set     = the distinct ids, sorted

mix64 is the splitmix64 finalizer; arithmetic is mod 2^64.
"""
from __future__ import annotations

M64 = (1 << 64) - 1
FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3
GOLDEN = 0x9E3779B97F4A7C15
WHITESPACE = b" \t\n\v\f\r"


def fnv1a64(data: bytes) -> int:
    h = FNV_OFFSET
    for b in data:
        h ^= b
        h = (h * FNV_PRIME) & M64
    return h


def mix64(z: int) -> int:
    """splitmix64 finalizer."""
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def splitmix64_stream(seed: int, n: int) -> list[int]:
    """The first n outputs of splitmix64 started at `seed` (for the known-answer pin)."""
    out, s = [], seed & M64
    for _ in range(n):
        s = (s + GOLDEN) & M64
        out.append(mix64(s))
    return out


def tokens(text: bytes) -> list[bytes]:
    out, cur = [], bytearray()
    for b in text:
        if b in WHITESPACE:
            if cur:
                out.append(bytes(cur))
                cur = bytearray()
        else:
            cur.append(b + 32 if 65 <= b <= 90 else b)
    if cur:
        out.append(bytes(cur))
    return out


def gram_id(toks: list[bytes], vocab_size: int, seed: int) -> int:
    h = seed & M64
    for t in toks:
        h = mix64((h + GOLDEN + fnv1a64(t)) & M64)
    return h % vocab_size


def shingle_text(text: bytes, w: int, vocab_size: int, seed: int) -> list[int]:
    """The sorted distinct shingle ids of one document."""
    toks = tokens(text)
    return sorted({gram_id(toks[i:i + w], vocab_size, seed) for i in range(len(toks) - w + 1)})


def shingle_docs(docs: list[bytes], w: int, vocab_size: int, seed: int):
    """CSR (offsets [n+1] uint64, ids uint32) of a document collection."""
    import numpy as np
    sets = [shingle_text(d, w, vocab_size, seed) for d in docs]
    offsets = np.zeros(len(sets) + 1, dtype=np.uint64)
    np.cumsum([len(s) for s in sets], out=offsets[1:])
    ids = np.array([x for s in sets for x in s], dtype=np.uint32)
    return offsets, ids
