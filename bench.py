#!/usr/bin/env python
"""bench.py -- the OPH / GOPH / HOPH hot path (SURVEY 8(a) rows a1-a3, a5-a8,
a10) on BASELINE.json's image-like workload (configs[2]: 10^6 sets x 4,096
queries, k = 512, the largest single-GPU config), timed on the device; rank 0
prints ONE JSON line.

A step, per GPU (rank r owns its own shard of the config's collection, set
IDs offset by r * N; the queries are the same on every rank):
  a1-a3  oph_build_sketches   OPH (k) + HOPH (1:1, k') sketches of the shard
  a5     query sketches (rank 0) + broadcast; query prep inside compare_*
  a6-a8  compare_full / compare_goph / compare_hoph (threshold hit lists)
  a10    one device->host read of the hit counts; hit lists gathered to
         rank 0 (N > 1) and sorted (topk_or_threshold_results)

value = 3 * Q * N_total / step time: query x set comparisons per second of the
three OPH-family methods the metric names (every pair is scored by each of
full OPH, GOPH and HOPH in a step).

The MinWise baseline (rows a4, a9: k permutations, then scoring) is timed as
its own leg right after, with the same K / W: `baseline_minwise` in the line,
and `speedup_vs_minwise` = the paper's headline comparison ("HOPH is
five to seven times faster than MinWise"), build + score and score only.

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
(one process per GPU, 127.0.0.1).  --dist-backend gloo stages the two
collectives through host memory, so N ranks can share one GPU (a test of the
N > 1 step; the numbers of such a run are not scaling numbers).
--scaling strong (scale config only) splits the 8 shards of the 10^7-set
collection over the ranks instead of giving each rank its own shard.

`--impl reference` times the CPU oracle (the reference arm of this tier) on a
bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "query×set sketch comparisons/sec (HOPH, GOPH, full OPH) + sketches/sec; % HBM peak"
UNIT = "comparisons/s"
CONFIG_NAMES = ["image-like", "text-like", "scale", "sweep-0.2", "sweep-0.5", "sweep-0.9", "tiny"]

# bounded CPU samples of each workload for the oracle legs (about 5-10 s of CPU work each)
CPU_SAMPLE = {"image-like": (300_000, 64), "text-like": (100_000, 64), "scale": (100_000, 64),
              "sweep-0.2": (100_000, 64), "sweep-0.5": (100_000, 64), "sweep-0.9": (100_000, 64),
              "tiny": (2000, 100)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- workloads
def concat_workloads(ws):
    """One collection from several shards (strong scaling: a rank owns several of the 8
    scale shards); queries from the first (they are the same in every shard)."""
    import dataclasses
    offs, ids, planted, base, nnz = [np.zeros(1, dtype=np.uint64)], [], [], 0, 0
    for w in ws:
        offs.append(w.offsets[1:] + np.uint64(nnz))
        ids.append(w.ids)
        pl = w.planted.copy()
        pl[:, 1] += base
        planted.append(pl)
        base += w.n_sets
        nnz += int(w.offsets[-1])
    return dataclasses.replace(ws[0], offsets=np.concatenate(offs), ids=np.concatenate(ids),
                               planted=np.concatenate(planted))


def make_workload(config: str, rank: int, world: int, scaling: str):
    """(workload of this rank, scan strategy, hit capacity per method, survivor-capacity
    limit).  Weak scaling: every rank scores the same queries against its own shard.
    Strategy: PROBE where background similarity is low (text-like law), BRUTE where every
    set shares bins with the queries (Zipf image words, the sweep's hub)."""
    import paper_1805_11254_b200 as og
    from workloads import gen_gpu, text_like, tiny
    if config == "scale":  # configs[3]: 8 shards x 1.25M sets, 16,384 queries, T = 0.8
        shards = range(rank, 8, world) if scaling == "strong" else [rank]
        w = concat_workloads([gen_gpu.scale_shard(shard=s) for s in shards])
        return w, og.OPH_STRATEGY_PROBE, 1 << 24, 1 << 28
    if scaling == "strong":
        raise SystemExit("--scaling strong applies to the scale config (the 8-shard collection) only")
    if config == "text-like":
        return text_like(shard=rank), og.OPH_STRATEGY_PROBE, 1 << 22, 1 << 28
    if config == "image-like":
        return gen_gpu.image_like(shard=rank), og.OPH_STRATEGY_BITMAP, 1 << 23, 1 << 28
    if config.startswith("sweep-"):
        # 256 of the 1,024 hub perturbations per step: at Jmax = 0.9 a quarter of all pairs are hits
        return (gen_gpu.sweep(float(config.split("-")[1]), shard=rank, n_queries=256), og.OPH_STRATEGY_AUTO,
                1 << 28, 1 << 28)
    if config == "tiny":
        return tiny(), og.OPH_STRATEGY_AUTO, 1 << 20, 1 << 24
    raise ValueError(config)


# --------------------------------------------------------------------------- oracle (CPU) legs
def cpu_sample_step(w, n_sets: int, n_q: int):
    """The OPH-family path on a bounded sample with the CPU oracle: OPH + HOPH
    sketches of n_sets sets and n_q queries, full / GOPH / HOPH scoring,
    threshold lists (the rows `value` counts)."""
    import oracle
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    offs = w.offsets[: n_sets + 1]
    qoffs = w.q_offsets[: n_q + 1]
    lay = oracle.hoph_layout(V, p["a"], p["b"], p["hoph_kprime"])
    F = oracle.oph_sketch(offs, w.ids, V, p["k"], seed)
    H = oracle.hoph_sketch(offs, w.ids, V, lay, p["hoph_kprime"], seed)
    QF = oracle.oph_sketch(qoffs, w.q_ids, V, p["k"], seed)
    QH = oracle.hoph_sketch(qoffs, w.q_ids, V, lay, p["hoph_kprime"], seed)
    kw = dict(t_num=p["t_num"], t_den=p["t_den"])
    r1 = oracle.compare_full(QF, F, groups=p["k"] // p["kprime"], **kw)
    r2 = oracle.compare_goph(QF, F, n=p["k"] // p["kprime"], kprime=p["kprime"], eps=p["eps"], **kw)
    r3 = oracle.compare_hoph(QH, H, L=len(lay), kprime=p["hoph_kprime"], a=p["a"], b=p["b"], eps=p["eps"], **kw)
    return sum(len(oracle.threshold_list(r)) for r in (r1, r2, r3))


def cpu_workload(config: str):
    """The workload the oracle legs sample: the same generator and seed as the GPU arm's
    rank 0 (image-like / sweep / scale are drawn with torch on the GPU)."""
    from workloads import text_like, tiny
    if config == "text-like":
        return text_like()
    if config == "tiny":
        return tiny()
    w, _, _, _ = make_workload(config, 0, 1, "weak")
    return w


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    w = cpu_workload(args.config)
    n_s, n_q = CPU_SAMPLE[args.config]
    n_s, n_q = min(n_s, w.n_sets), min(n_q, w.n_queries)
    for _ in range(args.warmup):
        cpu_sample_step(w, n_s, n_q)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu_sample_step(w, n_s, n_q)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = 3 * n_q * n_s / t
    sample = (f"{args.config}: first {n_s} of {w.n_sets} sets x first {n_q} of {w.n_queries} queries; the "
              f"OPH-family path (OPH/HOPH sketches of the sample, full/GOPH/HOPH scoring, threshold lists)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": args.config, "sample_sets": n_s, "sample_queries": n_q},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "cpu": cpu_model(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU arm
def profile_kernels(fn):
    """Kernel launches of fn() and their device times, from the CUDA profiler (CUPTI),
    untimed: (launch count, {kernel: [count, total us]})."""
    try:
        import torch
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        n = 0
        per = {}
        for e in prof.events():
            if getattr(e, "device_type", None) is not None and "CUDA" in str(e.device_type):
                nm = e.name
                if "memset" in nm.lower() or "memcpy" in nm.lower():
                    continue
                n += 1
                key = nm.split("(")[0].replace("void ", "").replace("ophgpu::", "")
                c = per.setdefault(key, [0, 0.0])
                c[0] += 1
                c[1] += float(e.device_time_total)
        return n, per
    except Exception:  # profiler unavailable: no claim
        return None, {}


def ubench_peaks():
    """Measured ALU / issue peaks (scripts/ubench.cu, committed under profiles/)."""
    p = os.path.join(ROOT, "profiles", "ubench_r02.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


def ncu_traffic(config: str):
    p = os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(config, {})
    return {}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1805_11254_b200 as og
    from paper_1805_11254_b200 import dist as odist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    og.build()
    og.lib()

    w, strategy, cap, surv_limit = make_workload(args.config, rank, world, args.scaling)
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    N, Q = w.n_sets, w.n_queries
    if args.scaling == "strong":
        # every rank owns several of the 8 shards: set IDs from the ranks' actual sizes
        sizes = [N]
        if world > 1:
            nt = torch.tensor([N], dtype=torch.int64, device="cuda")
            allv = [torch.zeros_like(nt) for _ in range(world)]
            odist.all_gather(allv, nt)
            sizes = [int(x.item()) for x in allv]
        N_total = sum(sizes)
        base = sum(sizes[:rank])
    else:
        N_total = N * world
        base = rank * N
    k, kp, hkp, mwk = p["k"], p["kprime"], p["hoph_kprime"], p["mw_k"]
    flat = og.flat_layout(V, k, kp)
    hier = og.oph_hier_layout_make(V, p["a"], p["b"], hkp)
    L = hier.L
    prm = og.params(p["t_num"], p["t_den"], p["eps"], strategy=strategy)
    # MinWise has no BITMAP join (its values span the universe per permutation): its register scan
    prm_mw = og.params(p["t_num"], p["t_den"], p["eps"],
                       strategy=og.OPH_STRATEGY_BRUTE if strategy == og.OPH_STRATEGY_BITMAP else strategy)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    # resident inputs
    sets = og.SetCollection.from_numpy(w.offsets, w.ids)
    qsets = og.SetCollection.from_numpy(w.q_offsets, w.q_ids)
    so, sh = og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier)
    qo, qh = og.oph_build_sketches(qsets, V, seed, flat=flat, hier=hier)
    mw = og.minwise_build_sketches(sets, V, seed, mwk) if not args.no_minwise else None
    qmw = og.minwise_build_sketches(qsets, V, seed, mwk) if not args.no_minwise else None
    counts = torch.zeros((4,), dtype=torch.int64, device="cuda")
    # termination-level histograms of the four scorings (include/ophgpu.h d_stop_hist), per step
    hists = torch.zeros((4, og.OPH_STOP_HIST_LEN), dtype=torch.int64, device="cuda")
    # (set, bin) rows gathered by the BITMAP pipeline scans per step (include/ophgpu.h d_bins_scanned):
    # the measured algorithmic work of full OPH's scan, which stops a set once no pair can reach T
    scanned = torch.zeros((4,), dtype=torch.int64, device="cuda")
    res = []
    for i in range(4):
        r = og.Results(cap)
        r.count = counts[i:i + 1]
        r.stop_hist = hists[i]
        r.bins_scanned = scanned[i:i + 1]
        res.append(r)
    surv_cap = min(((Q + 31) // 32) * 32 * N, surv_limit)
    ws = [og.Workspace() for _ in range(5)]
    outs = [og.Results(cap * (world if rank == 0 else 1)) for _ in range(4)]
    merged = [og.Results(cap * world) for _ in range(4)] if world > 1 else None
    hit_bytes = og.HIT_DTYPE.itemsize

    def mark(ev, i):
        if ev is not None:
            ev[i].record(stream)

    def select(idx, n4):
        """a10: gather (N > 1) and sort method idx's hit list; returns the list length on rank 0."""
        n = n4[idx]
        src = res[idx]
        if world > 1:
            allh, cnts = odist.gather_hits(res[idx].hits, n)
            n = int(sum(cnts))
            if rank != 0:
                return n
            merged[idx].hits[: allh.numel()].copy_(allh)
            src = merged[idx]
        og.topk_or_threshold_results(src, n, og.OPH_SELECT_THRESHOLD, outs[idx], ws=ws[4])
        return n

    nvtx = torch.cuda.nvtx

    def step(ev=None, sets=sets, qsets=qsets):
        """One OPH-family pass (rows a1-a3, a5-a8, a10); ev[i] marks phase boundaries; NVTX
        ranges name the phases (ncu --nvtx --nvtx-include "oph_step/")."""
        nvtx.range_push("oph_step")
        mark(ev, 0)
        counts[:3].zero_()
        hists[:3].zero_()
        scanned[:3].zero_()
        nvtx.range_push("build_oph_hoph")
        og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier, out_oph=so, out_hoph=sh)
        nvtx.range_pop()
        mark(ev, 1)
        nvtx.range_push("query_sketches")
        if rank == 0:
            og.oph_build_sketches(qsets, V, seed, flat=flat, hier=hier, out_oph=qo, out_hoph=qh)
        if world > 1:
            odist.broadcast_tensors([qo.values, qo.empty, qh.values, qh.empty])
        nvtx.range_pop()
        mark(ev, 2)
        nvtx.range_push("compare_full")
        og.compare_full(qo, so, flat, prm, res[0], set_id_base=base, ws=ws[0])
        nvtx.range_pop()
        mark(ev, 3)
        nvtx.range_push("compare_goph")
        og.compare_goph(qo, so, flat, prm, res[1], set_id_base=base, ws=ws[1], survivor_capacity=surv_cap)
        nvtx.range_pop()
        mark(ev, 4)
        nvtx.range_push("compare_hoph")
        og.compare_hoph(qh, sh, hier, prm, res[2], set_id_base=base, ws=ws[2], survivor_capacity=surv_cap)
        nvtx.range_pop()
        mark(ev, 5)
        nvtx.range_push("select")
        n4 = [int(x) for x in counts[:3].cpu()]  # one device->host read of the three hit counts
        assert max(n4) <= cap, f"hit buffer overflow {n4}"
        total = [select(i, n4) for i in range(3)]
        nvtx.range_pop()
        mark(ev, 6)
        nvtx.range_pop()
        return total

    def step_mw(ev=None, sets=sets, qsets=qsets):
        """One MinWise-baseline pass (rows a4, a9, a10)."""
        mark(ev, 0)
        counts[3:].zero_()
        hists[3:].zero_()
        og.minwise_build_sketches(sets, V, seed, mwk, out=mw)
        mark(ev, 1)
        if rank == 0:
            og.minwise_build_sketches(qsets, V, seed, mwk, out=qmw)
        if world > 1:
            odist.broadcast_tensors([qmw.values, qmw.flags])
        mark(ev, 2)
        og.compare_minwise(qmw, mw, prm_mw, res[3], set_id_base=base, ws=ws[3])
        mark(ev, 3)
        n = int(counts[3:].cpu()[0])
        assert n <= cap, f"hit buffer overflow {n}"
        tot = select(3, [0, 0, 0, n])
        mark(ev, 4)
        return tot

    phase_ev = [("build_oph_hoph", 0, 1), ("query_sketches_oph_hoph", 1, 2), ("compare_full", 2, 3),
                ("compare_goph", 3, 4), ("compare_hoph", 4, 5), ("select", 5, 6)]
    phase_mw = [("build_minwise", 0, 1), ("query_sketches_minwise", 1, 2), ("compare_minwise", 2, 3),
                ("select_minwise", 3, 4)]

    def timed(fn, K, n_ev, clocks=None):
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n_ev)] for _ in range(K)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if clocks is not None:
            clocks.start()
            time.sleep(0.3)
        t0.record(stream)
        out = None
        for i in range(K):
            out = fn(evs[i])
        t1.record(stream)
        torch.cuda.synchronize()
        clk = clocks.stop() if clocks is not None else None
        if world > 1:
            dist.barrier()
        ms = t0.elapsed_time(t1) / K
        if world > 1:
            ms = odist.max_over_ranks(ms, device="cuda")
        return ms, evs, out, clk

    # warm-up
    for _ in range(args.warmup):
        step()
        if mw is not None:
            step_mw()
    torch.cuda.synchronize()

    # per-phase kernel lists (CUPTI, untimed): launch counts and device times of one step
    phase_kernels = {}
    launches = None
    if not args.no_launch_count:
        calls = {
            "build_oph_hoph": lambda: og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier, out_oph=so,
                                                            out_hoph=sh),
            "compare_full": lambda: og.compare_full(qo, so, flat, prm, res[0], set_id_base=base, ws=ws[0]),
            "compare_goph": lambda: og.compare_goph(qo, so, flat, prm, res[1], set_id_base=base, ws=ws[1],
                                                    survivor_capacity=surv_cap),
            "compare_hoph": lambda: og.compare_hoph(qh, sh, hier, prm, res[2], set_id_base=base, ws=ws[2],
                                                    survivor_capacity=surv_cap),
        }
        for name, fn in calls.items():
            phase_kernels[name] = profile_kernels(fn)[1]
        launches, step_kernels = profile_kernels(step)
    else:
        step_kernels = {}

    # ---------------- CUDA graph of the step's device part (one process per GPU, no collective
    # inside): the OPH+HOPH builds and the three compare calls, enqueued through the C-ABI once
    # and replayed, so the host's per-call work (argument checks, planner, ~25 launches) leaves
    # the timed loop; the select (a device->host read of the hit counts sizes the sorts) stays
    # eager.  Phase times come from the eager pass; the graph's hit counts must equal it.
    graph, graph_note = None, "off (--no-graph)" if args.no_graph else "off (N > 1: the query broadcast)"

    def step_dev():
        counts[:3].zero_()
        hists[:3].zero_()
        scanned[:3].zero_()
        og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier, out_oph=so, out_hoph=sh)
        og.oph_build_sketches(qsets, V, seed, flat=flat, hier=hier, out_oph=qo, out_hoph=qh)
        og.compare_full(qo, so, flat, prm, res[0], set_id_base=base, ws=ws[0])
        og.compare_goph(qo, so, flat, prm, res[1], set_id_base=base, ws=ws[1], survivor_capacity=surv_cap)
        og.compare_hoph(qh, sh, hier, prm, res[2], set_id_base=base, ws=ws[2], survivor_capacity=surv_cap)

    def step_graph(ev=None):
        mark(ev, 0)
        graph.replay()
        mark(ev, 1)
        n4 = [int(x) for x in counts[:3].cpu()]
        assert max(n4) <= cap, f"hit buffer overflow {n4}"
        total = [select(i, n4) for i in range(3)]
        mark(ev, 2)
        return total

    # (capturable only without host synchronisation inside the calls: BITMAP, or survivor lists
    # large enough that PROBE's GOPH / HOPH need no optimistic pass -- include/ophgpu.h)
    no_sync = strategy == og.OPH_STRATEGY_BITMAP or ((Q + 31) // 32) * 32 * N <= surv_limit
    if world == 1 and not args.no_graph and not no_sync:
        graph_note = "off (PROBE survivor lists smaller than Q x N: the calls synchronise)"
    if world == 1 and not args.no_graph and no_sync:
        try:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="relaxed"):
                step_dev()
            torch.cuda.synchronize()
            graph, graph_note = g, "on: builds + compare_full / goph / hoph replayed as one CUDA graph; select eager"
        except Exception as e:  # (a capture failure falls back to the eager step, recorded in the line)
            graph, graph_note = None, f"off (capture failed: {type(e).__name__}: {str(e)[:120]})"
            torch.cuda.synchronize()

    # ---------------- timed region (OPH family): device inputs resident in HBM
    K = args.steps
    ms, evs, hits_last, clk = timed(step, K, 7, ClockSampler(dev))
    phase_ms = {n: statistics.mean(evs[i][a].elapsed_time(evs[i][b]) for i in range(K)) for n, a, b in phase_ev}
    hh = hists.cpu().numpy().copy()
    scanned_step = [int(x) for x in scanned.cpu()]  # (last eager step)
    ms_eager = ms
    if graph is not None:
        for _ in range(2):
            step_graph()
        ms_g, _, hits_g, clk_g = timed(step_graph, K, 3, ClockSampler(dev))
        assert hits_g == hits_last, f"graph replay hits {hits_g} != eager {hits_last}"
        assert (hists.cpu().numpy()[:3] == hh[:3]).all(), "graph replay histograms differ from the eager step"
        ms, clk = ms_g, clk_g

    # ---------------- the MinWise baseline leg, same K / W (not in `value`)
    mw_line = None
    if mw is not None:
        ms_mw, evs_mw, hits_mw, clk_mw = timed(step_mw, K, 5, ClockSampler(dev))
        ph_mw = {n: statistics.mean(evs_mw[i][a].elapsed_time(evs_mw[i][b]) for i in range(K)) for n, a, b in phase_mw}
        hh[3] = hists[3].cpu().numpy()
        e2e_oph = {m: phase_ms["build_oph_hoph"] + phase_ms["query_sketches_oph_hoph"] + phase_ms["compare_" + m]
                   for m in ("full", "goph", "hoph")}
        e2e_mw = ph_mw["build_minwise"] + ph_mw["query_sketches_minwise"] + ph_mw["compare_minwise"]
        mw_line = {
            "ms_per_step": ms_mw, "phase_ms": ph_mw, "hits": hits_mw,
            "comparisons_per_s": Q * N_total / (ms_mw / 1e3),
            "sketches_per_s": N_total / (ph_mw["build_minwise"] / 1e3),
            "clocks": clk_mw,
            "speedup_vs_minwise": {
                "definition": "MinWise (collection + query sketches, then scoring) time / the method's "
                              "(OPH+HOPH sketches of collection + queries, then its scoring); score_only: "
                              "compare_minwise / compare_<method>",
                "build_and_score": {m: e2e_mw / t for m, t in e2e_oph.items()},
                "score_only": {m: ph_mw["compare_minwise"] / phase_ms["compare_" + m] for m in ("full", "goph", "hoph")},
                "paper": "HOPH 5-7x faster than MinWise on its FS / ImageNet data, Java on one CPU (P:40, P:860)",
            },
        }

    # ---------------- e2e: the OPH-family step through the C-ABI with HOST (pinned) inputs and result
    # read-back.  Every step copies its inputs (collection CSR + query CSR) host->device and reads its
    # sorted hit lists back; the copies run on a copy stream into a second input buffer while the
    # previous step computes (double buffering), so they are inside the timed region but overlap compute.
    e2e = None
    if not args.no_e2e:
        host = [torch.from_numpy(w.offsets.astype(np.int64)).pin_memory(),
                torch.from_numpy(w.ids.view(np.int32)).pin_memory(),
                torch.from_numpy(w.q_offsets.astype(np.int64)).pin_memory(),
                torch.from_numpy(w.q_ids.view(np.int32)).pin_memory()]
        h2d = sum(t.numel() * t.element_size() for t in (host if rank == 0 else host[:2]))
        bufs = [(og.SetCollection(torch.empty_like(sets.offsets), torch.empty_like(sets.ids)),
                 og.SetCollection(torch.empty_like(qsets.offsets), torch.empty_like(qsets.ids))) for _ in range(2)]
        cstream = torch.cuda.Stream()
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]

        def enqueue_copy(j):
            b = bufs[j % 2]
            with torch.cuda.stream(cstream):
                if j >= 2:
                    cstream.wait_event(consumed[j % 2])
                b[0].offsets.copy_(host[0], non_blocking=True)
                b[0].ids.copy_(host[1], non_blocking=True)
                if rank == 0:
                    b[1].offsets.copy_(host[2], non_blocking=True)
                    b[1].ids.copy_(host[3], non_blocking=True)
                copied[j % 2].record(cstream)

        d2h = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        cstream.wait_event(e0)
        enqueue_copy(0)
        for i in range(K):
            stream.wait_event(copied[i % 2])
            if i + 1 < K:
                enqueue_copy(i + 1)
            tot = step(None, sets=bufs[i % 2][0], qsets=bufs[i % 2][1])
            consumed[i % 2].record(stream)
            d2h = 3 * 8
            if rank == 0:
                for j in range(3):
                    if tot[j]:
                        _ = outs[j].hits[: tot[j] * hit_bytes].cpu()
                        d2h += tot[j] * hit_bytes
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / K
        if world > 1:
            ems = odist.max_over_ranks(ems, device="cuda")
        e2e = {"value": 3 * Q * N_total / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ems,
               "note": "H2D of step i+1 inputs overlaps step i compute (copy stream, double buffer)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---------------- work saved by early termination: per method, the pairs
    # decided after each number of groups compared (the last step's histograms, this rank)
    term = {}
    bins_compared = {}
    for i, (m, gsize, gtot) in enumerate((("full", kp, k // kp), ("goph", kp, k // kp), ("hoph", hkp, L),
                                          ("minwise", mwk, 1))):
        h = hh[i]
        npairs = int(h.sum())
        if npairs == 0:
            continue
        groups = float((h * np.arange(len(h))).sum() / max(1, npairs))
        bins = mwk if m == "minwise" else groups * gsize
        bins_compared[m] = float((h * np.arange(len(h))).sum()) * gsize if m != "minwise" else npairs * mwk
        term[m] = {"pairs": npairs, "hist": {str(g): int(c) for g, c in enumerate(h) if c},
                   "mean_groups_compared": groups if m != "minwise" else None,
                   "mean_bins_compared": bins, "bins_total": (mwk if m == "minwise" else gtot * gsize)}

    # ---------------- roofline of the dominant hot-path kernel
    peaks, peak_src = load_peaks()
    ub = ubench_peaks()
    f_sm = peaks.get("sm_max_mhz", 1965.0) * 1e6
    hbm = peaks["hbm_gbs"] * 1e9
    nnz = int(w.offsets[-1])
    nw_k, nw_h = (k + 31) // 32, (L * hkp + 31) // 32
    g_l0 = og.plan_thresholds(og.OPH_METHOD_GOPH, k // kp, kp, p["t_num"], p["t_den"], p["eps"])[2]
    # BRUTE compare: 2 warp-instructions (ISETP + predicated IMAD) per 32 bin-compares -> the issue
    # ceiling is 16 bin-compares per SMSP per clock; the measured rate of that exact loop is in
    # profiles/ubench_r02.json (scripts/ubench.cu)
    issue_peak = 148 * 4 * 16 * f_sm
    issue_src = "derived: 148 SM x 4 SMSP x 16 bin-compares/clk (2 warp-instr per 32 compares) x sm_max_mhz"
    # (scripts/ubench.cu's stand-alone ISETP+IMAD loop reaches 1.04e13/s, LESS than scan_kernel itself
    # on the sweep configs (1.12e13/s): it is not a ceiling, so the derived one is the peak; the
    # microbenchmark's LOP3 / IMAD lane rates (1.86e13/s = one warp-instr per SMSP per clock) confirm it)
    if ub and ub.get("brute_compares_per_s"):
        issue_src += f"; scripts/ubench.cu compare loop: {ub['brute_compares_per_s']:.3e}/s (below the kernel: not used)"
    # algorithmic bytes / work per launch
    build_bytes = 4 * nnz + 8 * (N + 1) + 4 * N * (k + L * hkp) + 4 * N * (nw_k + nw_h)
    scan_bytes = {"compare_full": N * (4 * k + 4 * nw_k),
                  "compare_goph": N * (4 * g_l0 * kp + 4 * ((g_l0 * kp + 31) // 32)),
                  "compare_hoph": N * (4 * hkp + 4)}
    models = {}
    l2_src = "none measured"

    # BITMAP join (K7): per (set, bin, block of 2,048 queries) one 4-B entry of the value -> row
    # table and one 256-B row of query bits, gathered from the L2-resident block tables; peak =
    # the measured random 256-B row-gather rate from a 16-MB table (scripts/ubench.cu)
    def l2_peak_for(row_bytes):
        key = "gather_128B_rows_GBps" if row_bytes == 128 else "gather_256B_rows_GBps"
        return (ub or {}).get(key, {}).get(str(16 << 20))

    def model_for(kernel: str, phase: str):
        if kernel.startswith("bit_scan") or kernel.startswith("bit_pipe"):
            # blocks of 2,048 queries (256-B rows; bit_scan_kernel, the OPHGPU_BIT_QW=1 A/B: 1,024)
            qwords = 1 if kernel.startswith("bit_scan_kernel") else 2
            row = 128 * qwords
            m = phase.split("_")[1]
            bins = (bins_compared.get(m, Q * N * k) / Q) if m != "full" else N * k  # (set, bin) pairs scanned
            gathered = bins * -(-Q // (1024 * qwords)) * (row + 4)
            # the pipelined scans count the rows they gathered (d_bins_scanned, over all blocks):
            # measured work instead of the model (full OPH's exit, R32; GOPH's levels 1 .. l0 + 1)
            ph_i = {"full": 0, "goph": 1}.get(m)
            if kernel.startswith("bit_pipe") and ph_i is not None and scanned_step[ph_i] > 0:
                gathered = scanned_step[ph_i] * (row + 4)
            peak = l2_peak_for(row)
            nonlocal l2_src
            l2_src = (f"measured: scripts/ubench.cu random {row}-B row gathers, 16-MB table "
                      "(profiles/ubench_r02.json)" if peak else "none measured")
            return ("l2", gathered, (peak or float("nan")) * 1e9, "GB/s", 1e9,
                    f"bytes: one {row}-B query-bit row + one 4-B table entry per (set, bin compared, "
                    f"{1024 * qwords}-query block)")
        if kernel.startswith("build_kernel") or kernel.startswith("build_warp_kernel"):
            return ("hbm", build_bytes, hbm, "GB/s", 1e9, "bytes: CSR in + OPH/HOPH sketches and masks out")
        if kernel.startswith("join_kernel"):
            return ("hbm", scan_bytes[phase], hbm, "GB/s", 1e9, "bytes: the scanned collection bins, one pass")
        if kernel.startswith("scan_kernel") or kernel.startswith("levels_kernel"):
            m = phase.split("_")[1]
            work = bins_compared.get(m, Q * N * k) if m != "full" else Q * N * k
            return ("alu", work, issue_peak, "bin-compares/s", 1.0,
                    "work: (query, set, bin) equality tests the method needs (termination histograms)")
        return None

    dom, dom_phase, dom_us = None, None, -1.0
    for ph, kl in phase_kernels.items():
        for kn, (cnt, us) in kl.items():
            if us > dom_us:
                dom, dom_phase, dom_us = kn, ph, us
    roof = None
    if dom is not None:
        mdl = model_for(dom, dom_phase)
        ph_us = sum(v[1] for v in phase_kernels[dom_phase].values())
        if mdl is not None:
            bound, work, peak, unit, scale, what = mdl
            # the call's CUDA-event time in the timed region, times the kernel's share of the call's
            # device time (CUPTI of the same call): the call's other kernels (query prep) are excluded
            share = dom_us / ph_us if ph_us > 0 else 1.0
            t_kernel = phase_ms[dom_phase] / 1e3 * share
            launches_dom = phase_kernels[dom_phase][dom][0]
            ach = work / t_kernel
            tr = ncu_traffic(args.config).get(dom.split("<")[0])
            roof = {"kernel": dom, "phase": dom_phase, "bound": bound, "achieved": ach / scale, "peak": peak / scale,
                    "unit": unit, "frac": ach / peak, "traffic": tr, "launches_per_step": launches_dom,
                    "work_per_step": work, "work": what, "kernel_ms": t_kernel * 1e3,
                    "kernel_share_of_call": share,
                    "peak_source": {"hbm": peak_src, "l2": l2_src}.get(bound, issue_src),
                    "bin_compares_per_s": (Q * N * k if dom_phase == "compare_full" else
                                           bins_compared.get(dom_phase.split("_")[1], 0)) / t_kernel,
                    "step_share": t_kernel * 1e3 / ms}
    per_phase = {}
    for ph, byt in list(scan_bytes.items()) + [("build_oph_hoph", build_bytes)]:
        per_phase[ph] = {"ms": phase_ms[ph], "hbm_bytes": byt, "hbm_frac": byt / (phase_ms[ph] / 1e3) / hbm}

    # ---------------- quality vs exact Jaccard, untimed: every reported pair of the
    # last step is verified with exact_jaccard_pairs (precision); recall counts the planted pairs
    # whose realised J >= T (background pairs: a 100,000-pair random sample is verified too),
    # for both empty-bin modes (EitherEmpty = the timed run; JointEmpty re-scored)
    quality = None
    if not args.no_quality and getattr(w, "planted", None) is not None and len(w.planted):
        tn, td = p["t_num"], p["t_den"]
        pl = np.asarray(w.planted)
        truth = {(int(q), int(s_)) for q, s_, i_, u_ in pl if u_ and i_ * td >= tn * u_}

        def verify(qi, si):
            qa = torch.as_tensor(np.asarray(qi, dtype=np.int32), device="cuda")
            sa = torch.as_tensor(np.asarray(si, dtype=np.int32), device="cuda")
            it, un = og.exact_jaccard_pairs(qsets, sets, qa, sa)
            it, un = it.cpu().numpy().astype(np.int64), un.cpu().numpy().astype(np.int64)
            return (un > 0) & (it * td >= tn * un)

        def score(r, n):
            h = r.numpy(min(n, r.capacity))
            qi, si = h["query"].astype(np.int64), h["set_id"].astype(np.int64) - base
            good = verify(qi, si) if len(h) else np.zeros(0, bool)
            rep = set(zip(qi.tolist(), si.tolist()))
            return {"hits": int(len(h)), "precision": float(good.mean()) if len(h) else None,
                    "recall": len(rep & truth) / max(1, len(truth))}

        rng = np.random.default_rng(12345)
        bq, bs = rng.integers(0, Q, 100_000), rng.integers(0, N, 100_000)
        planted_pairs = {(int(q), int(s_)) for q, s_, _, _ in pl}
        keep = np.array([(int(a_), int(b_)) not in planted_pairs for a_, b_ in zip(bq, bs)], dtype=bool)
        bq, bs = bq[keep], bs[keep]
        bg_above = int(verify(bq, bs).sum())
        n4q = counts.cpu().numpy()
        methods = ("full", "goph", "hoph", "minwise") if mw is not None else ("full", "goph", "hoph")
        quality = {"T": f"{tn}/{td}", "true_pairs": len(truth),
                   "truth": "planted pairs with realised J >= T; background check: "
                            f"{bg_above} of {len(bq)} random non-planted (query, set) pairs have exact J >= T",
                   "either_empty": {m: score(res[i], int(n4q[i])) for i, m in enumerate(methods)}}
        prm_j = og.params(p["t_num"], p["t_den"], p["eps"], joint=True, strategy=strategy)
        jr = [og.Results(cap) for _ in range(3)]
        og.compare_full(qo, so, flat, prm_j, jr[0], set_id_base=base, ws=ws[0])
        og.compare_goph(qo, so, flat, prm_j, jr[1], set_id_base=base, ws=ws[1], survivor_capacity=surv_cap)
        og.compare_hoph(qh, sh, hier, prm_j, jr[2], set_id_base=base, ws=ws[2], survivor_capacity=surv_cap)
        quality["joint_empty"] = {m: score(jr[i], jr[i].n()) for i, m in enumerate(("full", "goph", "hoph"))}
        # the empty-aware GOPH rule (E1-E4): not part of the timed
        # step; its quality in both empty modes and device time per call
        variants = {}
        for joint, key in ((False, "either_empty"), (True, "joint_empty")):
            prm_e = og.params(p["t_num"], p["t_den"], p["eps"], joint=joint, strategy=prm_mw.strategy,
                              variant=og.OPH_VARIANT_EMPTY_AWARE)
            er = og.Results(cap, stop_hist=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            og.compare_goph(qo, so, flat, prm_e, er, set_id_base=base, ws=ws[1], survivor_capacity=surv_cap)
            e1.record()
            torch.cuda.synchronize()
            quality[key]["goph_empty_aware"] = score(er, er.n())
            h = er.hist().astype(np.float64)
            variants[key] = {"ms_per_call_with_histogram": e0.elapsed_time(e1),
                             "mean_bins_compared": float((h * np.arange(len(h))).sum() / max(1.0, h.sum()) * kp)}
        quality["goph_empty_aware_runs"] = variants

    # ---------------- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        n_s, n_q = CPU_SAMPLE[args.config]
        n_s, n_q = min(n_s, N), min(n_q, Q)
        t0 = time.perf_counter()
        cpu_sample_step(w, n_s, n_q)
        t = time.perf_counter() - t0
        cpu = {"value": 3 * n_q * n_s / t, "unit": UNIT, "cores": oracle.num_threads(), "cpu": cpu_model(),
               "kind": "oracle",
               "sample": f"{args.config}: first {n_s} sets x first {n_q} queries, the OPH-family path (OPH/HOPH "
                         f"sketches, full/GOPH/HOPH scoring, threshold lists), {t:.1f} s"}

    flush = (f"inputs larger than L2: CSR {4 * nnz / 1e6:.0f} MB + OPH/HOPH sketches "
             f"{4 * N * (k + L * hkp) / 1e9:.2f} GB per step")
    line = {
        "metric": METRIC, "value": 3 * Q * N_total / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": args.config, "sets_per_gpu": N, "sets_total": N_total, "queries": Q, "k": k,
                   "kprime": kp, "hoph_groups": L, "minwise_k": mwk, "T": f"{p['t_num']}/{p['t_den']}",
                   "epsilon": p["eps"], "parallelism": f"set-sharded x{world} ({args.dist_backend})",
                   "scan_strategy": ["auto", "brute", "probe", "bitmap"][strategy], "l2": flush},
        "value_definition": "3 * queries * sets_total / step time; a step = OPH+HOPH sketches of the collection "
                            "and the queries, full OPH + GOPH + HOPH threshold scoring of every pair, hit lists "
                            "gathered and sorted (MinWise: baseline_minwise)",
        "sketches_per_s": {"oph_hoph": N_total / (phase_ms["build_oph_hoph"] / 1e3)},
        "comparisons_per_s": {m: Q * N_total / (phase_ms["compare_" + m] / 1e3) for m in ("full", "goph", "hoph")},
        "phase_ms": phase_ms,
        "hits": hits_last,
        "roofline": roof,
        "phases": per_phase,
        "baseline_minwise": mw_line,
        "termination": term,
        "quality": quality,
        "device_us_per_step": {n: {"launches": v[0], "us": round(v[1], 1)} for n, v in sorted(
            step_kernels.items(), key=lambda kv: -kv[1][1])},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches * K if launches is not None else None,
        "clocks": clk,
        "timing": {"step": graph_note, "ms_per_step_eager": ms_eager,
                   "phase_ms": "eager step, CUDA events between the calls"},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="image-like", choices=CONFIG_NAMES,
                    help="workload (BASELINE.json configs); image-like (the largest single-GPU config) is the headline")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--no-minwise", action="store_true", help="skip the MinWise baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-quality", action="store_true", help="skip the precision/recall pass (untimed)")
    ap.add_argument("--no-launch-count", action="store_true", help="skip the CUPTI kernel lists (use under ncu)")
    ap.add_argument("--no-graph", action="store_true", help="time the eager step (no CUDA graph replay)")
    args = ap.parse_args()
    if args.steps < 1 or args.warmup < 0:
        ap.error("--steps >= 1, --warmup >= 0")
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        # one process per GPU: re-launch under torchrun (127.0.0.1 rendezvous)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
               *sys.argv[1:]]
        return subprocess.call(cmd)
    if ws_env is not None and int(ws_env) != args.gpus:
        print(f"bench.py: WORLD_SIZE={ws_env} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
