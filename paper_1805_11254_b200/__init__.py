"""B200-native OPH / GOPH / HOPH near-duplicate scoring (arxiv 1805.11254).

A thin ctypes binding over the C-ABI library `lib/libophgpu.so` declared in
`include/ophgpu.h`.  The functions below carry the C names and only
marshal arguments: they allocate output tensors with PyTorch (device memory,
streams) and pass raw device pointers.  Every step of the path runs in the
library's sm_100a kernels; there is no CPU fallback -- a missing library or
CUDA device raises.

Layout conventions: sketch matrices are
bin-major `[n_bins, ld]` uint32 (held in int32 tensors), `ld` = n_sets
rounded up to a multiple of 32; empty masks `[ceil(n_bins/32), ld]`.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Optional

import numpy as np

from .build import LIB, build  # noqa: F401

c_u32, c_u64, c_vp, c_dbl = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_double

OPH_OK, OPH_EINVAL, OPH_EINCOMPAT, OPH_EOVERFLOW, OPH_ECUDA, OPH_EAMBIGUOUS, OPH_ENOMEM = range(7)
OPH_PERM_KEYED, OPH_PERM_IDENTITY = 0, 1
OPH_EMPTY_EITHER, OPH_EMPTY_JOINT = 0, 1
OPH_RES_THRESHOLD, OPH_RES_DENSE = 0, 1
OPH_SELECT_THRESHOLD, OPH_SELECT_TOPK = 0, 1
OPH_METHOD_FULL, OPH_METHOD_GOPH, OPH_METHOD_HOPH, OPH_METHOD_MINWISE = range(4)
OPH_FLAG_UNDEFINED, OPH_FLAG_EARLY = 1, 2
OPH_STRATEGY_AUTO, OPH_STRATEGY_BRUTE, OPH_STRATEGY_PROBE, OPH_STRATEGY_BITMAP = 0, 1, 2, 3
OPH_VARIANT_PAPER, OPH_VARIANT_EMPTY_AWARE = 0, 1
OPH_EMPTY = 0xFFFFFFFF
MAX_GROUPS = 64

HIT_DTYPE = np.dtype([("query", "<u4"), ("set_id", "<u4"), ("n_mb", "<u2"), ("n_excl", "<u2"),
                      ("groups", "u1"), ("verdict", "u1"), ("flags", "u1"), ("pad", "u1"), ("estimate", "<f4")])
assert HIT_DTYPE.itemsize == 20


class oph_perm(ctypes.Structure):
    _fields_ = [("vocab_size", c_u64), ("seed", c_u64), ("kind", c_u32), ("pad", c_u32)]


class oph_flat_layout(ctypes.Structure):
    _fields_ = [("vocab_size", c_u64), ("k", c_u32), ("kprime", c_u32)]


class oph_hier_layout(ctypes.Structure):
    _fields_ = [("vocab_size", c_u64), ("a", c_u32), ("b", c_u32), ("kprime", c_u32), ("L", c_u32),
                ("start", c_u64 * MAX_GROUPS), ("len", c_u64 * MAX_GROUPS)]

    def groups(self):
        return [(int(self.start[i]), int(self.len[i])) for i in range(self.L)]


class oph_sets(ctypes.Structure):
    _fields_ = [("d_offsets", c_vp), ("d_ids", c_vp), ("n_sets", c_u64)]


class oph_sketches(ctypes.Structure):
    _fields_ = [("d_values", c_vp), ("d_empty", c_vp), ("d_flags", c_vp), ("n_sets", c_u64), ("ld", c_u64),
                ("n_bins", c_u32), ("pad", c_u32), ("seed", c_u64), ("vocab_size", c_u64)]


class oph_params(ctypes.Structure):
    _fields_ = [("t_num", c_u32), ("t_den", c_u32), ("epsilon", c_dbl), ("empty_mode", c_u32), ("strategy", c_u32),
                ("variant", c_u32)]


class oph_results(ctypes.Structure):
    _fields_ = [("d_hits", c_vp), ("capacity", c_u64), ("d_count", c_vp), ("mode", c_u32), ("pad", c_u32),
                ("d_stop_hist", c_vp), ("d_bins_scanned", c_vp)]


OPH_STOP_HIST_LEN = 65  # include/ophgpu.h: OPH_MAX_GROUPS + 1


class OphError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_string(status)} (status {status})")


_lib = None

# every symbol include/ophgpu.h declares
EXPORTS = ["oph_status_string", "oph_sketch_ld", "oph_hier_layout_make", "oph_build_sketches",
           "minwise_build_sketches", "oph_workspace_size", "oph_workspace_size_for", "compare_full", "compare_goph", "compare_hoph",
           "compare_minwise", "oph_select_workspace_size", "topk_or_threshold_results", "oph_plan_thresholds",
           "exact_jaccard_pairs", "shingle_workspace_size", "shingle_text", "oph_validate_sets"]


def lib():
    """Load libophgpu.so (no fallback: raises if it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} is missing; build it with `python -m paper_1805_11254_b200.build`")
        L = ctypes.CDLL(LIB)
        L.oph_status_string.restype = ctypes.c_char_p
        L.oph_status_string.argtypes = [ctypes.c_int]
        L.oph_sketch_ld.restype = c_u64
        L.oph_sketch_ld.argtypes = [c_u64]
        for name in EXPORTS[2:]:
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def status_string(s: int) -> str:
    return lib().oph_status_string(int(s)).decode()


def _check(status: int, what: str):
    if status != OPH_OK:
        raise OphError(status, what)


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1805_11254_b200 needs a CUDA device (B200 / sm_100a); there is no CPU path")
    return torch


def _stream(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return c_vp(s.cuda_stream)


def _on(stream):
    """Make `stream` current for the binding's own temporaries (outputs,
    default workspaces, zero-fills, count reads): they are then allocated,
    filled and released in the order of the kernels the call enqueues on that
    stream.  A caller-owned Workspace / Results must be usable on `stream`."""
    import contextlib
    if stream is None:
        return contextlib.nullcontext()
    return _torch().cuda.stream(stream)


def _ptr(t):
    return c_vp(t.data_ptr()) if t is not None else None


def sketch_ld(n_sets: int) -> int:
    return int(lib().oph_sketch_ld(c_u64(n_sets)))


# --------------------------------------------------------------------------- host helpers
def oph_hier_layout_make(vocab_size: int, a: int, b: int, kprime: int) -> oph_hier_layout:
    out = oph_hier_layout()
    _check(lib().oph_hier_layout_make(c_u64(vocab_size), c_u32(a), c_u32(b), c_u32(kprime), ctypes.byref(out)),
           "oph_hier_layout_make")
    return out


def flat_layout(vocab_size: int, k: int, kprime: int) -> oph_flat_layout:
    return oph_flat_layout(vocab_size, k, kprime)


def params(t_num: int, t_den: int, epsilon: float, joint: bool = False, strategy: int = 0,
           variant: int = 0) -> oph_params:
    """Filter parameters; variant = OPH_VARIANT_EMPTY_AWARE selects the empty-aware GOPH rule."""
    return oph_params(t_num, t_den, epsilon, OPH_EMPTY_JOINT if joint else OPH_EMPTY_EITHER, strategy, variant)


def plan_thresholds(method: int, nlev: int, kprime: int, t_num: int, t_den: int, epsilon: float, a: int = 1, b: int = 1):
    """The planner's compiled per-level thresholds (acc, rej), l0 and weights."""
    acc = (c_u64 * max(1, nlev))()
    rej = (ctypes.c_int64 * max(1, nlev))()
    w = (c_u64 * nlev)()
    l0 = c_u32()
    _check(lib().oph_plan_thresholds(c_u32(method), c_u32(nlev), c_u32(kprime), c_u32(a), c_u32(b), c_u32(t_num),
                                     c_u32(t_den), c_dbl(epsilon), acc, rej, ctypes.byref(l0), w),
           "oph_plan_thresholds")
    return [int(x) for x in acc[:nlev - 1]], [int(x) for x in rej[:nlev - 1]], int(l0.value), [int(x) for x in w]


# --------------------------------------------------------------------------- device data
@dataclasses.dataclass
class SetCollection:
    """CSR set collection on the device (offsets int64 [n+1], ids int32 [nnz] holding uint32)."""
    offsets: "object"
    ids: "object"

    @property
    def n_sets(self) -> int:
        return int(self.offsets.numel()) - 1

    def c(self) -> oph_sets:
        return oph_sets(_ptr(self.offsets), _ptr(self.ids), self.n_sets)

    @staticmethod
    def from_numpy(offsets: np.ndarray, ids: np.ndarray, device="cuda") -> "SetCollection":
        torch = _torch()
        off = torch.from_numpy(np.ascontiguousarray(offsets).astype(np.int64)).to(device)
        idt = torch.from_numpy(np.ascontiguousarray(ids).astype(np.uint32).view(np.int32)).to(device)
        return SetCollection(off, idt)


@dataclasses.dataclass
class Sketches:
    """Bin-major sketch matrix on the device plus its provenance."""
    values: "object"              # int32 [n_bins, ld] holding uint32
    empty: Optional["object"]     # int32 [ceil(n_bins/32), ld] or None (MinWise)
    flags: Optional["object"]     # uint8 [ld] (MinWise) or None
    n_sets: int
    n_bins: int
    seed: int
    vocab_size: int

    @property
    def ld(self) -> int:
        return int(self.values.shape[1])

    def c(self) -> oph_sketches:
        return oph_sketches(_ptr(self.values), _ptr(self.empty), _ptr(self.flags), self.n_sets, self.ld,
                            self.n_bins, 0, self.seed, self.vocab_size)

    def numpy(self) -> np.ndarray:
        """Set-major [n_sets, n_bins] uint32 copy (host)."""
        return self.values.cpu().numpy().view(np.uint32)[:, : self.n_sets].T.copy()

    def empty_numpy(self) -> np.ndarray:
        return self.empty.cpu().numpy().view(np.uint32)[:, : self.n_sets].T.copy()


def _alloc_sketch(n_bins: int, n_sets: int, with_empty: bool):
    torch = _torch()
    ld = sketch_ld(n_sets)
    vals = torch.empty((n_bins, ld), dtype=torch.int32, device="cuda")
    emp = torch.empty(((n_bins + 31) // 32, ld), dtype=torch.int32, device="cuda") if with_empty else None
    return vals, emp, ld


def _oph_build_sketches_impl(sets: SetCollection, vocab_size: int, seed: int, flat: Optional[oph_flat_layout] = None,
                       hier: Optional[oph_hier_layout] = None, identity: bool = False, stream=None,
                       out_oph: Optional[Sketches] = None, out_hoph: Optional[Sketches] = None):
    """OPH and/or HOPH sketches of every set (one psi evaluation per element).
    Returns (oph Sketches or None, hoph Sketches or None)."""
    perm = oph_perm(vocab_size, seed, OPH_PERM_IDENTITY if identity else OPH_PERM_KEYED, 0)
    n = sets.n_sets
    ld = sketch_ld(n)
    so = sh = None
    if flat is not None:
        so = out_oph
        if so is None:
            v, e, ld = _alloc_sketch(flat.k, n, True)
            so = Sketches(v, e, None, n, flat.k, seed, vocab_size)
    if hier is not None:
        sh = out_hoph
        if sh is None:
            v, e, ld = _alloc_sketch(hier.L * hier.kprime, n, True)
            sh = Sketches(v, e, None, n, hier.L * hier.kprime, seed, vocab_size)
    _check(lib().oph_build_sketches(
        ctypes.byref(sets.c()), ctypes.byref(perm),
        ctypes.byref(flat) if flat is not None else None, _ptr(so.values) if so else None, _ptr(so.empty) if so else None,
        ctypes.byref(hier) if hier is not None else None, _ptr(sh.values) if sh else None,
        _ptr(sh.empty) if sh else None, c_u64(ld), _stream(stream)), "oph_build_sketches")
    return so, sh


def oph_validate_sets(sets: SetCollection, vocab_size: int, stream=None):
    """The CSR input contract check (debug aid; synchronises): raises OphError(OPH_EINVAL)
    on a violation (ids not strictly increasing, an id >= vocab_size, offsets decreasing)."""
    with _on(stream):
        _check(lib().oph_validate_sets(ctypes.byref(sets.c()), c_u64(vocab_size), _stream(stream)),
               "oph_validate_sets")


def _minwise_build_sketches_impl(sets: SetCollection, vocab_size: int, seed: int, k: int, stream=None,
                           out: Optional[Sketches] = None) -> Sketches:
    torch = _torch()
    n = sets.n_sets
    if out is None:
        v, _, ld = _alloc_sketch(k, n, False)
        fl = torch.empty((ld,), dtype=torch.uint8, device="cuda")
        out = Sketches(v, None, fl, n, k, seed, vocab_size)
    _check(lib().minwise_build_sketches(ctypes.byref(sets.c()), c_u64(vocab_size), c_u64(seed), c_u32(k),
                                        _ptr(out.values), _ptr(out.flags), c_u64(out.ld), _stream(stream)),
           "minwise_build_sketches")
    return out


# --------------------------------------------------------------------------- results / workspace
class Results:
    """A result sink: `capacity` oph_hit records + a device counter."""

    def __init__(self, capacity: int, dense: bool = False, stop_hist: bool = False, bins_scanned: bool = False):
        torch = _torch()
        self.capacity = int(capacity)
        self.mode = OPH_RES_DENSE if dense else OPH_RES_THRESHOLD
        self.hits = torch.zeros((max(1, self.capacity) * HIT_DTYPE.itemsize,), dtype=torch.uint8, device="cuda")
        self.count = torch.zeros((1,), dtype=torch.int64, device="cuda")
        # termination-level histogram (include/ophgpu.h d_stop_hist), accumulated over calls
        self.stop_hist = torch.zeros((OPH_STOP_HIST_LEN,), dtype=torch.int64, device="cuda") if stop_hist else None
        # (set, bin) rows gathered by BITMAP scans (include/ophgpu.h d_bins_scanned), accumulated
        self.bins_scanned = torch.zeros((1,), dtype=torch.int64, device="cuda") if bins_scanned else None

    def reset(self):
        self.count.zero_()
        if self.stop_hist is not None:
            self.stop_hist.zero_()
        if self.bins_scanned is not None:
            self.bins_scanned.zero_()

    def c(self) -> oph_results:
        return oph_results(_ptr(self.hits), self.capacity, _ptr(self.count), self.mode, 0,
                           _ptr(self.stop_hist) if self.stop_hist is not None else None,
                           _ptr(self.bins_scanned) if getattr(self, "bins_scanned", None) is not None else None)

    def hist(self) -> np.ndarray:
        """The termination-level histogram (synchronises)."""
        return self.stop_hist.cpu().numpy().astype(np.uint64)

    def n(self) -> int:
        """Records reported (synchronises); may exceed capacity (truncation)."""
        return int(self.count.item())

    def numpy(self, n: Optional[int] = None) -> np.ndarray:
        if n is None:
            n = self.capacity if self.mode == OPH_RES_DENSE else min(self.n(), self.capacity)
        raw = self.hits[: n * HIT_DTYPE.itemsize].cpu().numpy()
        return raw.view(HIT_DTYPE).copy()


class Workspace:
    """A growable device scratch buffer."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int):
        torch = _torch()
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty((max(nbytes, 256),), dtype=torch.uint8, device="cuda")
        return self.buf


def oph_workspace_size(method: int, n_queries: int, n_sets: int, n_bins: int, survivor_capacity: int = 0) -> int:
    out = ctypes.c_size_t()
    _check(lib().oph_workspace_size(c_u32(method), c_u64(n_queries), c_u64(n_sets), c_u32(n_bins),
                                    c_u64(survivor_capacity), ctypes.byref(out)), "oph_workspace_size")
    return int(out.value)


def oph_workspace_size_for(method: int, q: Sketches, s: Sketches, prm: oph_params, survivor_capacity: int = 0) -> int:
    out = ctypes.c_size_t()
    _check(lib().oph_workspace_size_for(c_u32(method), ctypes.byref(q.c()), ctypes.byref(s.c()), ctypes.byref(prm),
                                        c_u64(survivor_capacity), ctypes.byref(out)), "oph_workspace_size_for")
    return int(out.value)


def _ws(ws, method, q: Sketches, s: Sketches, survivor_capacity, prm=None):
    if prm is not None:
        nbytes = oph_workspace_size_for(method, q, s, prm, survivor_capacity)
    else:
        nbytes = oph_workspace_size(method, q.n_sets, s.n_sets, q.n_bins, survivor_capacity)
    if ws is None:
        ws = Workspace()
    buf = ws.get(nbytes)
    return buf


def _compare_full_impl(q: Sketches, s: Sketches, layout: oph_flat_layout, prm: oph_params, res: Results,
                 set_id_base: int = 0, ws: Optional[Workspace] = None, stream=None):
    buf = _ws(ws, OPH_METHOD_FULL, q, s, 0, prm)
    _check(lib().compare_full(ctypes.byref(q.c()), ctypes.byref(s.c()), c_u32(set_id_base), ctypes.byref(layout),
                              ctypes.byref(prm), ctypes.byref(res.c()), _ptr(buf), ctypes.c_size_t(buf.numel()),
                              _stream(stream)), "compare_full")


def _compare_goph_impl(q: Sketches, s: Sketches, layout: oph_flat_layout, prm: oph_params, res: Results,
                 set_id_base: int = 0, ws: Optional[Workspace] = None, survivor_capacity: int = 0, stream=None):
    buf = _ws(ws, OPH_METHOD_GOPH, q, s, survivor_capacity, prm)
    _check(lib().compare_goph(ctypes.byref(q.c()), ctypes.byref(s.c()), c_u32(set_id_base), ctypes.byref(layout),
                              ctypes.byref(prm), ctypes.byref(res.c()), _ptr(buf), ctypes.c_size_t(buf.numel()),
                              _stream(stream)), "compare_goph")


def _compare_hoph_impl(q: Sketches, s: Sketches, layout: oph_hier_layout, prm: oph_params, res: Results,
                 set_id_base: int = 0, ws: Optional[Workspace] = None, survivor_capacity: int = 0, stream=None):
    buf = _ws(ws, OPH_METHOD_HOPH, q, s, survivor_capacity, prm)
    _check(lib().compare_hoph(ctypes.byref(q.c()), ctypes.byref(s.c()), c_u32(set_id_base), ctypes.byref(layout),
                              ctypes.byref(prm), ctypes.byref(res.c()), _ptr(buf), ctypes.c_size_t(buf.numel()),
                              _stream(stream)), "compare_hoph")


def _compare_minwise_impl(q: Sketches, s: Sketches, prm: oph_params, res: Results, set_id_base: int = 0,
                    ws: Optional[Workspace] = None, stream=None):
    buf = _ws(ws, OPH_METHOD_MINWISE, q, s, 0, prm)
    _check(lib().compare_minwise(ctypes.byref(q.c()), ctypes.byref(s.c()), c_u32(set_id_base), ctypes.byref(prm),
                                 ctypes.byref(res.c()), _ptr(buf), ctypes.c_size_t(buf.numel()), _stream(stream)),
           "compare_minwise")


def oph_select_workspace_size(n_in: int) -> int:
    out = ctypes.c_size_t()
    _check(lib().oph_select_workspace_size(c_u64(n_in), ctypes.byref(out)), "oph_select_workspace_size")
    return int(out.value)


def _exact_jaccard_pairs_impl(queries: SetCollection, sets: SetCollection, query_idx, set_idx, stream=None):
    """|Q_a n S_b| and |Q_a u S_b| for pairs (query_idx[i], set_idx[i]) (int32/uint32
    device tensors; set_idx local to `sets`) -> (inter, union) uint32-as-int32 tensors."""
    torch = _torch()
    n = int(query_idx.numel())
    inter = torch.zeros((max(1, n),), dtype=torch.int32, device="cuda")
    union = torch.zeros((max(1, n),), dtype=torch.int32, device="cuda")
    _check(lib().exact_jaccard_pairs(ctypes.byref(queries.c()), ctypes.byref(sets.c()), _ptr(query_idx),
                                     _ptr(set_idx), c_u64(n), _ptr(inter), _ptr(union), _stream(stream)),
           "exact_jaccard_pairs")
    return inter[:n], union[:n]


def _shingle_text_impl(text, doc_offsets, w: int, vocab_size: int, seed: int, ids_capacity: Optional[int] = None,
                 ws: Optional[Workspace] = None, stream=None) -> SetCollection:
    """Documents (uint8 device tensor of bytes + int64 device offsets [n_docs+1], offsets[0] = 0)
    -> their shingle sets as a CSR SetCollection (include/ophgpu.h shingle_text)."""
    torch = _torch()
    n_docs = int(doc_offsets.numel()) - 1
    n_bytes = int(text.numel())
    nb = ctypes.c_size_t()
    _check(lib().shingle_workspace_size(c_u64(n_bytes), c_u64(n_docs), ctypes.byref(nb)), "shingle_workspace_size")
    buf = (ws or Workspace()).get(nb.value)
    cap = ids_capacity if ids_capacity is not None else (n_bytes + n_docs) // 2 + 1
    offsets = torch.zeros((n_docs + 1,), dtype=torch.int64, device="cuda")
    ids = torch.zeros((max(1, cap),), dtype=torch.int32, device="cuda")
    n_ids = torch.zeros((1,), dtype=torch.int64, device="cuda")
    _check(lib().shingle_text(_ptr(text), _ptr(doc_offsets), c_u64(n_docs), c_u64(n_bytes), c_u32(w), c_u64(vocab_size),
                              c_u64(seed), _ptr(offsets), _ptr(ids), c_u64(cap), _ptr(n_ids), _ptr(buf),
                              ctypes.c_size_t(buf.numel()), _stream(stream)), "shingle_text")
    n = int(n_ids.item())
    if n > cap:
        raise OphError(OPH_EOVERFLOW, f"shingle_text: {n} ids > capacity {cap}")
    return SetCollection(offsets, ids[:n])


def _topk_or_threshold_results_impl(res_in: Results, n_in: int, mode: int, out: Results, topk: int = 0, k_bins: int = 0,
                              ws: Optional[Workspace] = None, stream=None):
    """Sort (threshold) or select per-query top-k from the first n_in records
    of res_in into out (out.count receives the number written)."""
    nbytes = oph_select_workspace_size(n_in)
    buf = (ws or Workspace()).get(nbytes)
    _check(lib().topk_or_threshold_results(_ptr(res_in.hits), c_u64(n_in), c_u32(mode), c_u32(topk), c_u32(k_bins),
                                           _ptr(out.hits), _ptr(out.count), _ptr(buf), ctypes.c_size_t(buf.numel()),
                                           _stream(stream)), "topk_or_threshold_results")


# --------------------------------------------------------------------------- stream-safe entry points
# Every public call runs with `stream` current (see _on): a caller passing a
# non-current stream gets temporaries ordered with the kernels on that stream.
def _with_stream(impl):
    import functools

    @functools.wraps(impl)
    def call(*args, stream=None, **kw):
        with _on(stream):
            return impl(*args, stream=stream, **kw)
    call.__name__ = call.__qualname__ = impl.__name__[1:-len("_impl")]
    return call


oph_build_sketches = _with_stream(_oph_build_sketches_impl)
minwise_build_sketches = _with_stream(_minwise_build_sketches_impl)
compare_full = _with_stream(_compare_full_impl)
compare_goph = _with_stream(_compare_goph_impl)
compare_hoph = _with_stream(_compare_hoph_impl)
compare_minwise = _with_stream(_compare_minwise_impl)
exact_jaccard_pairs = _with_stream(_exact_jaccard_pairs_impl)
shingle_text = _with_stream(_shingle_text_impl)
topk_or_threshold_results = _with_stream(_topk_or_threshold_results_impl)
