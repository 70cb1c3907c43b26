"""Seeded synthetic set collections shaped like the paper's workloads.

This module is INPUT DATA ONLY.  It holds none of the method's arithmetic
(no permutation, no binning, no sketch, no comparison): it draws sets of
integer feature IDs and planted near-duplicates, and both the CPU oracle
(`oracle/`) and the CUDA path (`paper_1805_11254_b200/`) consume the very same
CSR arrays it returns.

The paper's datasets -- the FS text corpus of NSFC proposals
and the 1M-image ImageNet SIFT subset -- are not available
here.  These generators stand in for them with the shapes BASELINE.json's
`configs` prescribe; the recipe of every config is restated in DESIGN.md
("Input recipe").

Planted duplicates follow SPEC.md `gen_pair`: a duplicate of a
query of size s keeps i = round(2sJ/(1+J)) random elements of the query and
adds s-i fresh elements that are not in the query, so its realised Jaccard is
exactly i/(2s-i); the realised value (not the target J) is recorded.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

U32 = np.uint32
U64 = np.uint64


@dataclasses.dataclass
class Workload:
    """One synthetic workload: a collection (CSR) plus a query batch (CSR)."""
    name: str
    vocab_size: int
    offsets: np.ndarray      # uint64 [n_sets+1]
    ids: np.ndarray          # uint32 [nnz], strictly increasing within a set
    q_offsets: np.ndarray    # uint64 [n_queries+1]
    q_ids: np.ndarray        # uint32 [q_nnz]
    planted: np.ndarray      # int64 [n_planted, 4]: (query, set_id, |q∩p|, |q∪p|)
    params: dict             # method parameters of the config (k, kprime, T, eps, ...)

    @property
    def n_sets(self) -> int:
        return len(self.offsets) - 1

    @property
    def n_queries(self) -> int:
        return len(self.q_offsets) - 1

    def set_ids(self, s: int) -> np.ndarray:
        return self.ids[int(self.offsets[s]):int(self.offsets[s + 1])]

    def query_ids(self, q: int) -> np.ndarray:
        return self.q_ids[int(self.q_offsets[q]):int(self.q_offsets[q + 1])]

    def slice_sets(self, lo: int, hi: int) -> "Workload":
        """Contiguous shard [lo, hi) of the collection (queries replicated)."""
        base = int(self.offsets[lo])
        offs = self.offsets[lo:hi + 1] - U64(base)
        ids = self.ids[base:int(self.offsets[hi])]
        keep = (self.planted[:, 1] >= lo) & (self.planted[:, 1] < hi)
        planted = self.planted[keep].copy()
        planted[:, 1] -= lo
        return dataclasses.replace(self, offsets=offs, ids=ids, planted=planted)


# --------------------------------------------------------------------------
# element samplers (ids in [0, V))
# --------------------------------------------------------------------------
def _uniform_sampler(V: int):
    def draw(rng, n):
        return rng.integers(0, V, size=n, dtype=np.uint64)
    return draw


def _zipf_sampler(V: int, s: float):
    """Word id = Zipf rank - 1, P(rank r) proportional to r^-s over [1, V]."""
    w = np.arange(1, V + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]

    def draw(rng, n):
        u = rng.random(n)
        return np.minimum(np.searchsorted(cdf, u, side="right"), V - 1).astype(np.uint64)
    return draw


def _csr_from_sorted_keys(keys: np.ndarray, n_sets: int):
    sets = (keys >> U64(32)).astype(np.int64)
    ids = (keys & U64(0xFFFFFFFF)).astype(U32)
    counts = np.bincount(sets, minlength=n_sets)
    offsets = np.zeros(n_sets + 1, dtype=U64)
    np.cumsum(counts, out=offsets[1:])
    return offsets, ids


def sample_sets(rng, sizes: np.ndarray, V: int, draw) -> tuple[np.ndarray, np.ndarray]:
    """Draw len(sizes) sets of distinct ids; set i has exactly sizes[i] ids
    (sizes are clipped to V).  Returns CSR (offsets uint64, ids uint32)."""
    assert V <= 2 ** 32
    sizes = np.minimum(np.asarray(sizes, dtype=np.int64), V)
    n = len(sizes)

    def sorted_unique(a):
        a.sort()
        if len(a) < 2:
            return a
        keep = np.empty(len(a), dtype=bool)
        keep[0] = True
        np.not_equal(a[1:], a[:-1], out=keep[1:])
        return a[keep]

    # rejection sampling: draw exactly the deficit of every set, drop repeats, repeat
    owner = np.repeat(np.arange(n, dtype=U64), sizes)
    keys = sorted_unique((owner << U64(32)) | draw(rng, int(sizes.sum())))
    for _ in range(10_000):
        have = np.bincount((keys >> U64(32)).astype(np.int64), minlength=n)
        need = sizes - have
        if not need.any():
            break
        deficient = need > 0
        own_all = (keys >> U64(32)).astype(np.int64)
        in_def = deficient[own_all]
        owner = np.repeat(np.arange(n, dtype=U64), need)
        sub = sorted_unique(np.concatenate([keys[in_def], (owner << U64(32)) | draw(rng, int(need.sum()))]))
        keys = np.concatenate([keys[~in_def], sub])
        keys.sort()
    else:
        raise RuntimeError("sample_sets: could not fill sets (V too small?)")
    return _csr_from_sorted_keys(keys, n)


def plant_duplicate(rng, q: np.ndarray, J: float, V: int, draw) -> tuple[np.ndarray, int, int]:
    """SPEC gen_pair relative to an existing query q: keep
    i = round(2sJ/(1+J)) elements of q, add s-i fresh ones not in q."""
    s = len(q)
    i = int(round(2 * s * J / (1 + J)))
    i = max(0, min(i, s))
    keep = rng.choice(q, size=i, replace=False) if i > 0 else np.zeros(0, dtype=q.dtype)
    fresh: set[int] = set()
    qset = set(int(x) for x in q)
    while len(fresh) < s - i:
        for x in draw(rng, 2 * (s - i - len(fresh)) + 4):
            x = int(x)
            if x not in qset and x not in fresh:
                fresh.add(x)
                if len(fresh) == s - i:
                    break
    out = np.sort(np.concatenate([keep.astype(np.int64), np.fromiter(fresh, dtype=np.int64, count=len(fresh))]))
    return out.astype(U32), i, 2 * s - i


def _assemble(rng, name, V, bg_off, bg_ids, n_sets, planted_sets, q_off, q_ids, planted_meta, params):
    """Place planted sets at random set IDs among the background sets."""
    n_pl = len(planted_sets)
    slots = rng.permutation(n_sets)
    pl_slot = np.sort(slots[:n_pl])
    perm_pl = rng.permutation(n_pl)            # which planted set goes to which slot
    sizes = np.zeros(n_sets, dtype=np.int64)
    is_pl = np.zeros(n_sets, dtype=bool)
    is_pl[pl_slot] = True
    bg_sizes = np.diff(bg_off.astype(np.int64))
    sizes[~is_pl] = bg_sizes
    src_of_slot = {}
    for j, slot in enumerate(pl_slot):
        p = perm_pl[j]
        src_of_slot[int(slot)] = p
        sizes[slot] = len(planted_sets[p])
    offsets = np.zeros(n_sets + 1, dtype=U64)
    np.cumsum(sizes, out=offsets[1:])
    ids = np.empty(int(offsets[-1]), dtype=U32)
    # background sets, in order, into the non-planted slots
    bg_slots = np.nonzero(~is_pl)[0]
    # vectorised copy: destination index for each background id
    dst_start = offsets[:-1][bg_slots].astype(np.int64)
    lens = bg_sizes
    rel = np.arange(len(bg_ids), dtype=np.int64) - np.repeat(bg_off[:-1].astype(np.int64), lens)
    ids[np.repeat(dst_start, lens) + rel] = bg_ids
    meta = []
    for slot, p in src_of_slot.items():
        a, b = int(offsets[slot]), int(offsets[slot + 1])
        ids[a:b] = planted_sets[p]
        qi, inter, union = planted_meta[p]
        meta.append((qi, slot, inter, union))
    meta.sort()
    return Workload(name, V, offsets, ids, q_off, q_ids,
                    np.array(meta, dtype=np.int64).reshape(-1, 4), params)


# --------------------------------------------------------------------------
# the five BASELINE.json configs
# --------------------------------------------------------------------------
def tiny(seed: int = 1) -> Workload:
    """configs[0]: 2,000 sets over D=2^16, sizes U{50..300}, 100 queries each
    with 5 planted near-duplicates at J in {0.5,0.7,0.8,0.9,0.95}; k=64."""
    rng = np.random.default_rng(seed)
    V = 2 ** 16
    draw = _uniform_sampler(V)
    nq, n_sets = 100, 2000
    Js = [0.5, 0.7, 0.8, 0.9, 0.95]
    q_off, q_ids = sample_sets(rng, rng.integers(50, 301, size=nq), V, draw)
    planted_sets, meta = [], []
    for q in range(nq):
        qv = q_ids[int(q_off[q]):int(q_off[q + 1])]
        for J in Js:
            p, inter, union = plant_duplicate(rng, qv, J, V, draw)
            planted_sets.append(p)
            meta.append((q, inter, union))
    n_bg = n_sets - len(planted_sets)
    bg_off, bg_ids = sample_sets(rng, rng.integers(50, 301, size=n_bg), V, draw)
    params = dict(k=64, kprime=16, a=1, b=1, hoph_kprime=16, t_num=7, t_den=10,
                  eps=1e-4, mw_k=64, perm_seed=0x5EED0001)
    return _assemble(rng, "tiny", V, bg_off, bg_ids, n_sets, planted_sets, q_off, q_ids, meta, params)


def _lognormal_sizes(rng, n, mean=400.0, sigma=0.8):
    # mean 400 => mu = ln 400 - sigma^2/2 (the exp(mu)=400 reading is flagged in DESIGN.md)
    mu = math.log(mean) - sigma * sigma / 2
    return np.maximum(1, np.rint(rng.lognormal(mu, sigma, size=n))).astype(np.int64)


def text_like(seed: int = 2, n_sets: int = 200_000, n_queries: int = 1000,
              planted_frac: float = 0.01, shard: int = 0) -> Workload:
    """configs[1]: 200,000 shingle sets over 2^32, sizes lognormal(mean 400,
    sigma 0.8), 1,000 queries, 1% of the sets planted duplicates at
    J ~ U[0.6, 0.98]; k=256.

    The query batch depends on `seed` only; the collection on (seed, shard),
    so shard r of a multi-GPU run is an independent text-like collection of
    n_sets sets with its own planted duplicates of the SAME queries."""
    V = 2 ** 32
    draw = _uniform_sampler(V)
    rq = np.random.default_rng(seed)
    q_off, q_ids = sample_sets(rq, _lognormal_sizes(rq, n_queries), V, draw)
    rng = np.random.default_rng([seed, shard])
    n_pl = int(round(planted_frac * n_sets))
    planted_sets, meta = [], []
    for j in range(n_pl):
        q = (j + shard * n_pl) % n_queries
        qv = q_ids[int(q_off[q]):int(q_off[q + 1])]
        p, inter, union = plant_duplicate(rng, qv, float(rng.uniform(0.6, 0.98)), V, draw)
        planted_sets.append(p)
        meta.append((q, inter, union))
    bg_off, bg_ids = sample_sets(rng, _lognormal_sizes(rng, n_sets - n_pl), V, draw)
    params = dict(k=256, kprime=32, a=1, b=1, hoph_kprime=32, t_num=7, t_den=10,
                  eps=1e-4, mw_k=256, perm_seed=0x5EED0002)
    return _assemble(rng, "text-like", V, bg_off, bg_ids, n_sets, planted_sets, q_off, q_ids, meta, params)


def image_like(seed: int = 3, n_sets: int = 1_000_000, n_queries: int = 4096,
               planted_per_query: int = 4) -> Workload:
    """configs[2]: bag-of-visual-words, 1M sets over 2^20, Poisson(800) words
    per set drawn without replacement with Zipf(1.1) frequencies, 4,096
    queries with planted duplicates at J ~ U[0.5, 0.95]; k=512, k'=32."""
    rng = np.random.default_rng(seed)
    V = 2 ** 20
    draw = _zipf_sampler(V, 1.1)
    q_off, q_ids = sample_sets(rng, np.maximum(1, rng.poisson(800, size=n_queries)), V, draw)
    planted_sets, meta = [], []
    for q in range(n_queries):
        qv = q_ids[int(q_off[q]):int(q_off[q + 1])]
        for _ in range(planted_per_query):
            p, inter, union = plant_duplicate(rng, qv, float(rng.uniform(0.5, 0.95)), V, draw)
            planted_sets.append(p)
            meta.append((q, inter, union))
    bg_off, bg_ids = sample_sets(rng, np.maximum(1, rng.poisson(800, size=n_sets - len(planted_sets))), V, draw)
    params = dict(k=512, kprime=32, a=1, b=1, hoph_kprime=32, t_num=7, t_den=10,
                  eps=1e-4, mw_k=512, perm_seed=0x5EED0003)
    return _assemble(rng, "image-like", V, bg_off, bg_ids, n_sets, planted_sets, q_off, q_ids, meta, params)


CONFIGS = {"tiny": tiny, "text-like": text_like, "image-like": image_like}


def uniform_pair(rng, s: int, J: float, V: int):
    """Two sets of size s with |A∩B| = round(2sJ/(1+J)) (SPEC gen_pair)."""
    draw = _uniform_sampler(V)
    off, ids = sample_sets(rng, np.array([s]), V, draw)
    a = ids
    b, inter, union = plant_duplicate(rng, a, J, V, draw)
    return a, b, inter, union


def make_csr(sets) -> tuple[np.ndarray, np.ndarray]:
    """CSR from a list of id iterables (sorted + deduplicated here)."""
    arrs = [np.unique(np.asarray(list(s), dtype=np.int64)) for s in sets]
    offsets = np.zeros(len(arrs) + 1, dtype=U64)
    np.cumsum([len(a) for a in arrs], out=offsets[1:])
    ids = np.concatenate(arrs).astype(U32) if arrs and offsets[-1] > 0 else np.zeros(0, dtype=U32)
    return offsets, ids
