"""Seeded synthetic workloads at BASELINE.json's full sizes, drawn on the GPU.

INPUT DATA ONLY, like gen.py: no permutation, binning, sketch or comparison.
The numpy generators in gen.py are too slow at 10^6 - 10^7 sets, so the same
recipes are drawn here with torch on a CUDA device
and returned as host numpy CSR arrays; the oracle and the CUDA path consume
the very same arrays.  Deterministic for a given seed (torch's counter-based
CUDA generator).

* image-like (configs[2]): 10^6 sets over 2^20, Poisson(800) distinct words
  drawn without replacement with Zipf(1.1) weights (= i.i.d. Zipf draws with
  repeats discarded), 4,096 queries, 4 planted duplicates each at J ~ U[0.5,0.95].
* sweep (configs[4]): 2x10^6 sets over 2^20 (uniform ids), a hub H of
  Poisson(800) words; 1,024 queries are J = 0.98 perturbations of H; every
  collection set is built against H at J ~ U(0, Jmax) (SPEC gen_pair, equal
  sizes |H|), so every (query, set) pair sees the target distribution.
* scale (configs[3]) per-GPU shard: text-like law, 1.25x10^6 sets, 16,384
  queries, 1% planted at J ~ U[0.6, 0.98].
"""
from __future__ import annotations

import math

import numpy as np

from .gen import Workload, _assemble, _lognormal_sizes, _uniform_sampler, _zipf_sampler, plant_duplicate

U32, U64 = np.uint32, np.uint64


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("gen_gpu needs a CUDA device")
    return torch


def _distinct_first(torch, vals, sizes, V):
    """Row r of vals [R, M] (int64 ids < V): its first sizes[r] distinct values
    in order of first appearance.  Returns (row, value) pairs sorted by
    (row, value), or None if some row has fewer distinct values."""
    R, M = vals.shape
    dev = vals.device
    row = torch.arange(R, device=dev, dtype=torch.int64).unsqueeze(1).expand(R, M)
    pos = torch.arange(M, device=dev, dtype=torch.int64).unsqueeze(0).expand(R, M)
    key = (row * V + vals) * M + pos
    key, _ = torch.sort(key.reshape(-1))
    rv = key // M
    first = torch.ones_like(rv, dtype=torch.bool)
    first[1:] = rv[1:] != rv[:-1]
    rv, p = rv[first], key[first] % M
    r = rv // V
    # order the first occurrences of each row by position, keep the first sizes[r]
    k2, order = torch.sort(r * M + p)
    r, rv = r[order], rv[order]
    counts = torch.bincount(r, minlength=R)
    if bool((counts < sizes).any()):
        return None
    start = torch.zeros(R + 1, device=dev, dtype=torch.int64)
    start[1:] = torch.cumsum(counts, 0)
    rank = torch.arange(r.numel(), device=dev, dtype=torch.int64) - start[r]
    keep = rank < sizes[r]
    out, _ = torch.sort(rv[keep])  # (row, value) order: row * V + value
    return out


def _csr(torch, parts, n_sets, V):
    keys = torch.cat(parts)
    rows = keys // V
    ids = (keys % V).to(torch.int64)
    counts = torch.bincount(rows, minlength=n_sets)
    offsets = np.zeros(n_sets + 1, dtype=U64)
    np.cumsum(counts.cpu().numpy(), out=offsets[1:])
    return offsets, ids.cpu().numpy().astype(U32)


def sample_sets_gpu(gen, sizes: np.ndarray, V: int, draw, chunk: int = 16384):
    """CSR of len(sizes) sets of distinct ids; draw(gen, shape) -> int64 ids < V
    (i.i.d.); a set takes the first sizes[r] distinct draws."""
    torch = _torch()
    sizes = np.minimum(np.asarray(sizes, dtype=np.int64), V)
    n = len(sizes)
    parts = []
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        sz = torch.from_numpy(sizes[c0:c1]).cuda()
        mult = 1.25
        while True:
            M = int(max(8, math.ceil(mult * int(sz.max()) + 8)))
            sel = _distinct_first(torch, draw(gen, (c1 - c0, M)), sz, V)
            if sel is not None:
                break
            mult *= 2
        parts.append(sel + c0 * V)
    return _csr(torch, parts, n, V)


def _uniform_draw(V):
    def draw(gen, shape):
        torch = _torch()
        return torch.randint(0, V, shape, generator=gen, device="cuda", dtype=torch.int64)
    return draw


def _zipf_draw(V, s):
    torch = _torch()
    w = torch.arange(1, V + 1, device="cuda", dtype=torch.float64) ** (-s)
    cdf = torch.cumsum(w, 0)
    cdf /= cdf[-1].clone()

    def draw(gen, shape):
        u = torch.rand(shape, generator=gen, device="cuda", dtype=torch.float64)
        return torch.clamp(torch.searchsorted(cdf, u, right=True), max=V - 1).to(torch.int64)
    return draw


def image_like(seed: int = 3, n_sets: int = 1_000_000, n_queries: int = 4096, planted_per_query: int = 4,
               shard: int = 0) -> Workload:
    """The queries depend on `seed` only; the collection (with its planted
    duplicates of those queries) on (seed, shard)."""
    torch = _torch()
    V = 2 ** 20
    qgen = torch.Generator(device="cuda")
    qgen.manual_seed(seed)
    rq = np.random.default_rng(seed)
    zd = _zipf_draw(V, 1.1)
    q_off, q_ids = sample_sets_gpu(qgen, np.maximum(1, rq.poisson(800, size=n_queries)), V, zd)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed * 1000 + 7 + shard)
    rng = np.random.default_rng([seed, shard])
    cpu_draw = _zipf_sampler(V, 1.1)
    planted_sets, meta = [], []
    for q in range(n_queries):
        qv = q_ids[int(q_off[q]):int(q_off[q + 1])]
        for _ in range(planted_per_query):
            p, inter, union = plant_duplicate(rng, qv, float(rng.uniform(0.5, 0.95)), V, cpu_draw)
            planted_sets.append(p)
            meta.append((q, inter, union))
    bg_off, bg_ids = sample_sets_gpu(gen, np.maximum(1, rng.poisson(800, size=n_sets - len(planted_sets))), V, zd)
    params = dict(k=512, kprime=32, a=1, b=1, hoph_kprime=32, t_num=7, t_den=10,
                  eps=1e-4, mw_k=512, perm_seed=0x5EED0003, strategy="brute")
    return _assemble(rng, "image-like", V, bg_off, bg_ids, n_sets, planted_sets, q_off, q_ids, meta, params)


def sweep(jmax: float, seed: int = 5, n_sets: int = 2_000_000, n_queries: int = 1024, chunk: int = 65536,
          shard: int = 0) -> Workload:
    """configs[4] at one Jmax: every set is a gen_pair duplicate of the hub H at J ~ U(0, Jmax).
    The hub and the queries depend on (seed, Jmax); the collection also on shard."""
    torch = _torch()
    V = 2 ** 20
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed * 1000 + int(round(jmax * 100)))
    rng = np.random.default_rng([seed, int(round(jmax * 100))])
    draw = _uniform_draw(V)
    h_off, H = sample_sets_gpu(gen, np.array([max(2, rng.poisson(800))]), V, draw)
    if shard:
        gen.manual_seed(seed * 1000 + int(round(jmax * 100)) + 100003 * shard)
    s = len(H)
    cpu_draw = _uniform_sampler(V)
    qsets, meta_q = [], []
    for _ in range(n_queries):
        qv, _, _ = plant_duplicate(rng, H, 0.98, V, cpu_draw)
        qsets.append(qv)
    q_off = np.zeros(n_queries + 1, dtype=U64)
    np.cumsum([len(x) for x in qsets], out=q_off[1:])
    q_ids = np.concatenate(qsets).astype(U32)
    Hg = torch.from_numpy(H.astype(np.int64)).cuda()
    inH = torch.zeros(V, dtype=torch.bool, device="cuda")
    inH[Hg] = True
    J = torch.rand(n_sets, generator=gen, device="cuda", dtype=torch.float64) * jmax
    i_keep = torch.round(2 * s * J / (1 + J)).to(torch.int64).clamp(0, s)
    parts = []
    for c0 in range(0, n_sets, chunk):
        c1 = min(n_sets, c0 + chunk)
        R = c1 - c0
        ik = i_keep[c0:c1]
        # kept: the first i elements of a random permutation of H
        perm = torch.argsort(torch.rand((R, s), generator=gen, device="cuda"), dim=1)
        kept = Hg[perm]
        kmask = torch.arange(s, device="cuda").unsqueeze(0) < ik.unsqueeze(1)
        # fresh: s - i distinct ids not in H
        need = s - ik
        mult = 1.25
        while True:
            M = int(math.ceil(mult * int(need.max()) + 8))
            cand = draw(gen, (R, M))
            cand = torch.where(inH[cand], torch.full_like(cand, -1), cand)
            # push rejected candidates to the end with distinct negative placeholders
            sel = _distinct_first_masked(torch, cand, need, V)
            if sel is not None:
                break
            mult *= 2
        rows_k = torch.arange(R, device="cuda").unsqueeze(1).expand(R, s)[kmask]
        keys = torch.cat([rows_k * V + kept[kmask], sel])
        keys, _ = torch.sort(keys)
        parts.append(keys + c0 * V)
    off, ids = _csr(torch, parts, n_sets, V)
    params = dict(k=512, kprime=32, a=1, b=1, hoph_kprime=32, t_num=7, t_den=10,
                  eps=1e-4, mw_k=512, perm_seed=0x5EED0005, jmax=jmax, strategy="auto")
    # realised J of every pair (query, set) is not recorded (all pairs are "planted")
    return Workload(f"sweep-{jmax}", V, off, ids, q_off, q_ids, np.zeros((0, 4), dtype=np.int64), params)


def _distinct_first_masked(torch, cand, need, V):
    """Like _distinct_first, ignoring entries < 0 (rejected candidates)."""
    R, M = cand.shape
    valid = cand >= 0
    big = torch.where(valid, cand, torch.full_like(cand, V))  # rejected -> value V (sorted last)
    row = torch.arange(R, device=cand.device, dtype=torch.int64).unsqueeze(1).expand(R, M)
    pos = torch.arange(M, device=cand.device, dtype=torch.int64).unsqueeze(0).expand(R, M)
    key = (row * (V + 1) + big) * M + pos
    key, _ = torch.sort(key.reshape(-1))
    rv = key // M
    first = torch.ones_like(rv, dtype=torch.bool)
    first[1:] = rv[1:] != rv[:-1]
    v = rv % (V + 1)
    first &= v < V
    rv, p = rv[first], key[first] % M
    r = rv // (V + 1)
    v = rv % (V + 1)
    _, order = torch.sort(r * M + p)
    r, v = r[order], v[order]
    counts = torch.bincount(r, minlength=R)
    if bool((counts < need).any()):
        return None
    start = torch.zeros(R + 1, device=cand.device, dtype=torch.int64)
    start[1:] = torch.cumsum(counts, 0)
    rank = torch.arange(r.numel(), device=cand.device, dtype=torch.int64) - start[r]
    keep = rank < need[r]
    return r[keep] * V + v[keep]


def scale_shard(shard: int = 0, seed: int = 4, n_sets: int = 1_250_000, n_queries: int = 16384,
                planted_frac: float = 0.01) -> Workload:
    """configs[3], one of the 8 per-GPU shards of 10^7 text-like sets (T = 8/10)."""
    torch = _torch()
    V = 2 ** 32
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed * 100 + shard)
    rq = np.random.default_rng(seed)
    draw = _uniform_draw(V)
    qgen = torch.Generator(device="cuda")
    qgen.manual_seed(seed)
    q_off, q_ids = sample_sets_gpu(qgen, _lognormal_sizes(rq, n_queries), V, draw)
    rng = np.random.default_rng([seed, shard])
    n_pl = int(round(planted_frac * n_sets))
    cpu_draw = _uniform_sampler(V)
    planted_sets, meta = [], []
    for j in range(n_pl):
        q = (j + shard * n_pl) % n_queries
        qv = q_ids[int(q_off[q]):int(q_off[q + 1])]
        p, inter, union = plant_duplicate(rng, qv, float(rng.uniform(0.6, 0.98)), V, cpu_draw)
        planted_sets.append(p)
        meta.append((q, inter, union))
    bg_off, bg_ids = sample_sets_gpu(gen, _lognormal_sizes(rng, n_sets - n_pl), V, draw, chunk=8192)
    params = dict(k=256, kprime=32, a=1, b=1, hoph_kprime=32, t_num=8, t_den=10,
                  eps=1e-4, mw_k=256, perm_seed=0x5EED0004, strategy="auto")
    return _assemble(rng, "scale", V, bg_off, bg_ids, n_sets, planted_sets, q_off, q_ids, meta, params)
