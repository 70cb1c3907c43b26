#!/usr/bin/env python
"""bench.py -- one step of the whole OPH/GOPH/HOPH hot path (SURVEY 8(a) rows
a1-a10) on the text-like workload (BASELINE.json configs[1]), timed on the
device; prints ONE JSON line (rank 0).

A step, per GPU (rank r owns a text-like shard of 200,000 sets, set IDs
offset by r*200,000; the 1,000 queries are the same on every rank):
  a1-a3  oph_build_sketches     OPH (k=256) + HOPH (1:1, k'=32, L=27) of the shard
  a4     minwise_build_sketches MinWise (k=256) of the shard
  a5     query sketches (rank 0) + NCCL broadcast; query prep inside compare_*
  a6-a9  compare_full / compare_goph / compare_hoph / compare_minwise (threshold)
  a10    hit lists gathered to rank 0 and sorted (topk_or_threshold_results)

value = 3 * Q * N_total / step time: query x set comparisons per second of
the three OPH-family methods the metric names (every pair is scored by each
of full OPH, GOPH and HOPH in a step; MinWise and the sketch builds are
inside the timed step but not counted).

`--impl reference` times the CPU oracle (the reference arm of this tier) on
a bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
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

# CPU sample of the workload for the oracle legs (about 10 s of CPU work)
CPU_SAMPLE_SETS = 20_000
CPU_SAMPLE_QUERIES = 32


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


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


# --------------------------------------------------------------------------- oracle (CPU) legs
def cpu_sample_step(w, n_sets: int, n_q: int):
    """The whole path on a bounded sample, with the CPU oracle: sketches of
    n_sets sets and n_q queries, the four comparisons, threshold lists."""
    import oracle
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    offs = w.offsets[: n_sets + 1]
    qoffs = w.q_offsets[: n_q + 1]
    lay = oracle.hoph_layout(V, p["a"], p["b"], p["hoph_kprime"])
    F = oracle.oph_sketch(offs, w.ids, V, p["k"], seed)
    H = oracle.hoph_sketch(offs, w.ids, V, lay, p["hoph_kprime"], seed)
    MW, fl = oracle.minwise_sketch(offs, w.ids, V, p["mw_k"], seed)
    QF = oracle.oph_sketch(qoffs, w.q_ids, V, p["k"], seed)
    QH = oracle.hoph_sketch(qoffs, w.q_ids, V, lay, p["hoph_kprime"], seed)
    QMW, qfl = oracle.minwise_sketch(qoffs, w.q_ids, V, p["mw_k"], seed)
    kw = dict(t_num=p["t_num"], t_den=p["t_den"])
    r1 = oracle.compare_full(QF, F, groups=p["k"] // p["kprime"], **kw)
    r2 = oracle.compare_goph(QF, F, n=p["k"] // p["kprime"], kprime=p["kprime"], eps=p["eps"], **kw)
    r3 = oracle.compare_hoph(QH, H, L=len(lay), kprime=p["hoph_kprime"], a=p["a"], b=p["b"], eps=p["eps"], **kw)
    r4 = oracle.compare_minwise(QMW, qfl, MW, fl, **kw)
    return sum(len(oracle.threshold_list(r)) for r in (r1, r2, r3, r4))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    from workloads import text_like
    oracle.build()
    w = text_like()
    n_s, n_q = CPU_SAMPLE_SETS, CPU_SAMPLE_QUERIES
    for _ in range(args.warmup):
        cpu_sample_step(w, n_s, n_q)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu_sample_step(w, n_s, n_q)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = 3 * n_q * n_s / t
    sample = (f"text-like: first {n_s} of 200,000 sets x first {n_q} of 1,000 queries; whole path "
              f"(OPH/HOPH/MinWise sketches of the sample, full/GOPH/HOPH/MinWise scoring, threshold lists)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": "text-like", "sample_sets": n_s, "sample_queries": n_q},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU arm
CONFIG_NAMES = ["text-like", "image-like", "scale", "sweep-0.2", "sweep-0.5", "sweep-0.9", "tiny"]


def make_workload(config: str, rank: int):
    """(workload of this rank's shard, scan strategy, hit capacity per method,
    survivor-capacity limit).  Every rank scores the same queries against its
    own independent shard (weak scaling).  Strategy: PROBE where background
    similarity is low (text-like law), BRUTE where every set shares bins with
    the queries (Zipf image words, the sweep's hub)."""
    import paper_1805_11254_b200 as og
    from workloads import gen_gpu, text_like, tiny
    if config == "text-like":
        return text_like(shard=rank), og.OPH_STRATEGY_PROBE, 1 << 22, 1 << 28
    if config == "scale":  # configs[3]: 8 shards x 1.25M sets, 16,384 queries, T = 0.8
        return gen_gpu.scale_shard(shard=rank), og.OPH_STRATEGY_PROBE, 1 << 23, 1 << 28
    if config == "image-like":
        return gen_gpu.image_like(shard=rank), og.OPH_STRATEGY_BRUTE, 1 << 23, 1 << 28
    if config.startswith("sweep-"):
        # 256 of the 1,024 hub perturbations per step: at Jmax = 0.9 a quarter of all pairs are hits
        return (gen_gpu.sweep(float(config.split("-")[1]), shard=rank, n_queries=256), og.OPH_STRATEGY_BRUTE,
                1 << 28, 1 << 28)
    if config == "tiny":
        return tiny(), og.OPH_STRATEGY_AUTO, 1 << 20, 1 << 24
    raise ValueError(config)


def count_launches(step_fn):
    """Kernel launches of one step and their device times, from the CUDA profiler
    (CUPTI) over one extra, untimed step: (launch count, {kernel: [count, total us]})."""
    try:
        import torch
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step_fn()
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


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1805_11254_b200 as og
    from paper_1805_11254_b200 import dist as odist
    from workloads import text_like

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    og.build()
    og.lib()

    w, strategy, cap, surv_limit = make_workload(args.config, rank)
    p = w.params
    V, seed = w.vocab_size, p["perm_seed"]
    N, Q = w.n_sets, w.n_queries
    N_total = N * world
    base = rank * N
    k, kp, hkp, mwk = p["k"], p["kprime"], p["hoph_kprime"], p["mw_k"]
    flat = og.flat_layout(V, k, kp)
    hier = og.oph_hier_layout_make(V, p["a"], p["b"], hkp)
    L = hier.L
    prm = og.params(p["t_num"], p["t_den"], p["eps"], strategy=strategy)
    # the OPH family runs on a high-priority stream; the MinWise baseline (one long ALU-bound
    # kernel of short CTAs) on a normal-priority side stream fills the SMs around it
    lo_prio, hi_prio = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") \
        else (0, -1)
    stream = torch.cuda.Stream(priority=hi_prio)
    torch.cuda.set_stream(stream)

    # resident inputs
    sets = og.SetCollection.from_numpy(w.offsets, w.ids)
    qsets = og.SetCollection.from_numpy(w.q_offsets, w.q_ids)
    so, sh = og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier)
    mw = og.minwise_build_sketches(sets, V, seed, mwk)
    qo, qh = og.oph_build_sketches(qsets, V, seed, flat=flat, hier=hier)
    qmw = og.minwise_build_sketches(qsets, V, seed, mwk)
    counts = torch.zeros((4,), dtype=torch.int64, device="cuda")
    # termination-level histograms of the four scorings (include/ophgpu.h d_stop_hist), per step
    hists = torch.zeros((4, og.OPH_STOP_HIST_LEN), dtype=torch.int64, device="cuda")
    res = []
    for i in range(4):
        r = og.Results(cap)
        r.count = counts[i:i + 1]
        r.stop_hist = hists[i]
        res.append(r)
    surv_cap = min(((Q + 31) // 32) * 32 * N, surv_limit)
    ws = [og.Workspace() for _ in range(5)]
    outs = [og.Results(cap * (world if rank == 0 else 1)) for _ in range(4)]
    merged = [og.Results(cap * world) for _ in range(4)] if world > 1 else None

    side_stream = torch.cuda.Stream(priority=lo_prio)  # MinWise (the baseline) beside the OPH family

    def step(ev=None, inputs=None, sets=sets, qsets=qsets, serial=False):
        """One pass of rows a1-a10.  Stream `stream`: OPH/HOPH build, query
        sketches, full OPH / GOPH / HOPH; stream `side`: the MinWise build and
        scoring (ALU-bound) overlapping the OPH family (memory/latency-bound).
        ev[j] marks phase boundaries on the stream that runs the phase.
        serial=True runs everything on one stream (per-kernel timing)."""
        side = stream if serial else side_stream

        def mark(i, st=stream):
            if ev is not None:
                ev[i].record(st)
        mark(0)
        counts.zero_()
        hists.zero_()
        fork = torch.cuda.Event()
        fork.record(stream)
        side.wait_event(fork)
        qmw_ready = torch.cuda.Event()
        # ---- side stream: a4 MinWise build (collection; the queries' on the main stream, which
        # is idle meanwhile, so the side stream's critical path is the collection build), a9
        with torch.cuda.stream(side):
            mark(9, side)
            og.minwise_build_sketches(sets, V, seed, mwk, out=mw)
            mark(10, side)
        if not serial:
            if rank == 0:
                og.minwise_build_sketches(qsets, V, seed, mwk, out=qmw)
            if world > 1:
                odist.broadcast_tensors([qmw.values, qmw.flags])
            qmw_ready.record(stream)
        with torch.cuda.stream(side):
            if serial:
                if rank == 0:
                    og.minwise_build_sketches(qsets, V, seed, mwk, out=qmw)
                if world > 1:
                    odist.broadcast_tensors([qmw.values, qmw.flags])
            else:
                side.wait_event(qmw_ready)
            mark(11, side)
            og.compare_minwise(qmw, mw, prm, res[3], set_id_base=base, ws=ws[3])
            mark(12, side)
        # ---- main stream: a1-a3 OPH+HOPH build, a5 queries, a6-a8 scoring
        mark(8)
        og.oph_build_sketches(sets, V, seed, flat=flat, hier=hier, out_oph=so, out_hoph=sh)
        mark(1)
        if rank == 0:
            og.oph_build_sketches(qsets, V, seed, flat=flat, hier=hier, out_oph=qo, out_hoph=qh)
        if world > 1:
            odist.broadcast_tensors([qo.values, qo.empty, qh.values, qh.empty])
        mark(2)
        og.compare_full(qo, so, flat, prm, res[0], set_id_base=base, ws=ws[0])
        mark(3)
        og.compare_goph(qo, so, flat, prm, res[1], set_id_base=base, ws=ws[1], survivor_capacity=surv_cap)
        mark(4)
        og.compare_hoph(qh, sh, hier, prm, res[2], set_id_base=base, ws=ws[2], survivor_capacity=surv_cap)
        mark(5)
        # ---- a10 for the OPH family while the MinWise side stream is still busy (one GPU:
        # nothing to gather): read their three hit counts (syncs this stream only) and sort
        early = world == 1 and not serial
        if early:
            n3 = [int(x) for x in counts[:3].cpu()]
            assert max(n3) <= cap, f"hit buffer overflow {n3}"
            for i in range(3):
                og.topk_or_threshold_results(res[i], n3[i], og.OPH_SELECT_THRESHOLD, outs[i], ws=ws[4])
        join = torch.cuda.Event()
        join.record(side)
        stream.wait_event(join)
        mark(6)
        # ---- a10: gather (N > 1) and sort the (remaining) hit lists
        n4 = [int(x) for x in counts.cpu()]  # one device->host read of the four hit counts
        assert max(n4) <= cap, f"hit buffer overflow {n4}"
        total = []
        for i in range(4):
            src, n = res[i], n4[i]
            if early and i < 3:
                total.append(n)
                continue
            if world > 1:
                allh, cnts = odist.gather_hits(res[i].hits, n4[i])
                n = int(sum(cnts))
                if rank != 0:
                    continue
                merged[i].hits[: allh.numel()].copy_(allh)
                src = merged[i]
            if rank == 0:
                og.topk_or_threshold_results(src, n, og.OPH_SELECT_THRESHOLD, outs[i], ws=ws[4])
                total.append(n)
        mark(7)
        return total

    # phases: (name, start event, end event); 0..7 on the main stream, 9..12 on the side stream
    phase_ev = [("build_oph_hoph", 8, 1),("query_sketches_oph_hoph", 1, 2), ("compare_full", 2, 3),
                ("compare_goph", 3, 4), ("compare_hoph", 4, 5), ("join_minwise", 5, 6), ("select", 6, 7),
                ("build_minwise", 9, 10), ("query_sketches_minwise", 10, 11), ("compare_minwise", 11, 12)]

    # warm-up (also JIT-free: the .so is prebuilt)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # (the profiled step runs every call on one stream, so per-kernel device times are not
    # inflated by the MinWise side stream sharing the SMs)
    launches, kernel_us = (None, {}) if args.no_launch_count else count_launches(lambda: step(serial=True))

    # ---------------- timed region: device inputs resident in HBM
    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(13)] for _ in range(K)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    t_start.record(stream)
    hits_last = None
    for i in range(K):
        hits_last = step(evs[i])
    t_end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end) / K
    if world > 1:
        ms = odist.max_over_ranks(ms, device="cuda")
    phase_ms_concurrent = {n: statistics.mean(evs[i][a].elapsed_time(evs[i][b]) for i in range(K))
                           for n, a, b in phase_ev}

    # ---------------- per-kernel timing: the same K steps with every call on one stream, so each
    # call's CUDA-event time is its own duration (the rooflines below use these)
    evs_s = [[torch.cuda.Event(enable_timing=True) for _ in range(13)] for _ in range(K)]
    ts0, ts1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ts0.record(stream)
    for i in range(K):
        step(evs_s[i], serial=True)
    ts1.record(stream)
    torch.cuda.synchronize()
    ms_serial = ts0.elapsed_time(ts1) / K
    phase_ms = {n: statistics.mean(evs_s[i][a].elapsed_time(evs_s[i][b]) for i in range(K)) for n, a, b in phase_ev}

    # ---------------- e2e: same step through the C-ABI with HOST (pinned) inputs and result read-back.
    # Every step copies its inputs (collection CSR + query CSR) host->device and reads its sorted hit
    # lists back; the copies run on a copy stream into a second input buffer while the previous step
    # computes (double buffering), so they are inside the timed region but overlap compute.
    e2e = None
    if not args.no_e2e:
        host = [torch.from_numpy(w.offsets.astype(np.int64)).pin_memory(),
                torch.from_numpy(w.ids.view(np.int32)).pin_memory(),
                torch.from_numpy(w.q_offsets.astype(np.int64)).pin_memory(),
                torch.from_numpy(w.q_ids.view(np.int32)).pin_memory()]
        h2d = sum(t.numel() * t.element_size() for t in host)
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
            d2h = 4 * 8
            if rank == 0:
                for j in range(4):
                    n = tot[j]
                    if n:
                        _ = outs[j].hits[: n * 20].cpu()
                        d2h += n * 20
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

    # ---------------- roofline of the dominant kernel
    peaks, peak_src = load_peaks()
    f_sm = peaks.get("sm_max_mhz", 1965.0) * 1e6
    # ALU pipe (IADD3/LOP3/SHF/min): 16 lanes/clk/SMSP (B300_MICROARCH "rt_SMSP=2"), 148 SM x 4 SMSP;
    # one psi evaluation + running min is 9.5 ALU-pipe lane-ops at both widths (the SASS of
    # minwise_kernel: 5 LOP3 + 4 SHF + half a 3-input VIMNMX3)
    alu_lanes = 148 * 4 * 16 * f_sm
    w_bits = max(1, (V - 1).bit_length())
    psi_ops = 9.5
    psi_peak = alu_lanes / psi_ops
    hbm = peaks["hbm_gbs"] * 1e9
    nnz = int(w.offsets[-1])
    nw_k, nw_h = (k + 31) // 32, (L * hkp + 31) // 32
    g_l0 = og.plan_thresholds(og.OPH_METHOD_GOPH, k // kp, kp, p["t_num"], p["t_den"], p["eps"])[2]
    # algorithmic bytes per launch: inputs read once + outputs written once
    by = {
        "build_oph_hoph": 4 * nnz + 8 * (N + 1) + 4 * N * (k + L * hkp) + 4 * N * (nw_k + nw_h),
        "compare_full": N * (4 * k + 4 * nw_k),
        "compare_goph": N * (4 * g_l0 * kp + 4 * ((g_l0 * kp + 31) // 32)),
        "compare_hoph": N * (4 * hkp + 4),
        "compare_minwise": N * (4 * mwk + 1),
    }
    kern = {n: ("hbm", b / (phase_ms[n] / 1e3) / 1e9, hbm / 1e9, "GB/s", b) for n, b in by.items()}
    kern["build_minwise"] = ("alu", nnz * mwk / (phase_ms["build_minwise"] / 1e3), psi_peak, "psi-evals/s", None)
    traffic = {}
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f)
    dom = max(kern, key=lambda n: phase_ms[n])
    b, a_, pk, u, _ = kern[dom]
    roof = {"kernel": dom, "bound": b, "achieved": a_, "peak": pk, "unit": u, "frac": a_ / pk,
            "traffic": traffic.get(dom), "peak_source": peak_src if b == "hbm" else
            f"derived: 148 SM x 4 SMSP x 16 ALU lanes x sm_max_mhz / {psi_ops} ALU ops per psi (DESIGN.md)"}
    per_kernel = {n: {"ms": phase_ms[n], "bound": v[0], "achieved": v[1], "peak": v[2], "unit": v[3],
                      "frac": v[1] / v[2], "bytes": v[4]} for n, v in kern.items()}
    # the PROBE collection scans on their own (CUPTI device time of the join kernels over the
    # untimed profiled step): algorithmic bytes = one stream of the scanned bins per pass of
    # <= 4096 queries (full + GOPH prefix + HOPH group 1; MinWise separately)
    scan = {}
    passes = -(-Q // 4096)
    for name, mw_flag, byt in (("oph_family", "false", by["compare_full"] + by["compare_goph"] + by["compare_hoph"]),
                               ("minwise", "true", by["compare_minwise"])):
        hit = [v for kname, v in kernel_us.items() if kname.startswith(f"join_kernel<{mw_flag}")]
        if hit:
            us = sum(v[1] for v in hit)
            scan[name] = {"kernel": f"join_kernel<{mw_flag}, ...>", "launches": sum(v[0] for v in hit), "us": us,
                          "bytes": byt * passes, "achieved": byt * passes / (us / 1e6) / 1e9, "peak": hbm / 1e9,
                          "unit": "GB/s", "frac": byt * passes / (us / 1e6) / hbm}

    # ---------------- work saved by early termination: per method, the pairs
    # decided after each number of groups compared (the last step's histograms, this rank)
    hh = hists.cpu().numpy()
    term = {}
    for i, (m, gsize, gtot) in enumerate((("full", kp, k // kp), ("goph", kp, k // kp), ("hoph", hkp, L),
                                          ("minwise", mwk, 1))):
        h = hh[i]
        npairs = int(h.sum())
        groups = float((h * np.arange(len(h))).sum() / max(1, npairs))
        bins = mwk if m == "minwise" else groups * gsize
        term[m] = {"pairs": npairs, "hist": {str(g): int(c) for g, c in enumerate(h) if c},
                   "mean_groups_compared": groups if m != "minwise" else None,
                   "mean_bins_compared": bins, "bins_total": (mwk if m == "minwise" else gtot * gsize)}

    # ---------------- quality vs exact Jaccard, untimed: every reported pair of the
    # last step is verified with exact_jaccard_pairs (precision); recall counts the planted pairs
    # whose realised J >= T (background pairs are random sets: a 100,000-pair random sample is
    # verified too), for both empty-bin modes (EitherEmpty = the timed run; JointEmpty re-scored)
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
        quality = {"T": f"{tn}/{td}", "true_pairs": len(truth),
                   "truth": "planted pairs with realised J >= T; background check: "
                            f"{bg_above} of {len(bq)} random non-planted (query, set) pairs have exact J >= T",
                   "either_empty": {m: score(res[i], int(n4q[i])) for i, m in enumerate(("full", "goph", "hoph",
                                                                                          "minwise"))}}
        prm_j = og.params(p["t_num"], p["t_den"], p["eps"], joint=True, strategy=strategy)
        jr = [og.Results(cap) for _ in range(3)]
        og.compare_full(qo, so, flat, prm_j, jr[0], set_id_base=base, ws=ws[0])
        og.compare_goph(qo, so, flat, prm_j, jr[1], set_id_base=base, ws=ws[1], survivor_capacity=surv_cap)
        og.compare_hoph(qh, sh, hier, prm_j, jr[2], set_id_base=base, ws=ws[2], survivor_capacity=surv_cap)
        quality["joint_empty"] = {m: score(jr[i], jr[i].n()) for i, m in enumerate(("full", "goph", "hoph"))}
        # the empty-aware GOPH rule (E1-E4): not part of the timed
        # step; its quality in both empty modes, device time per call and termination histogram
        variants = {}
        for joint, key in ((False, "either_empty"), (True, "joint_empty")):
            prm_e = og.params(p["t_num"], p["t_den"], p["eps"], joint=joint, variant=og.OPH_VARIANT_EMPTY_AWARE)
            er = og.Results(cap, stop_hist=True)
            og.compare_goph(qo, so, flat, prm_e, er, set_id_base=base, ws=ws[1])
            torch.cuda.synchronize()
            quality[key]["goph_empty_aware"] = score(er, er.n())
            h = er.hist().astype(np.float64)
            # timed as a user calls it for a hit list: no histogram, so AUTO takes the join and
            # decides only the listed pairs (E5); with the histogram every pair's stop
            # group is needed and the register scan runs
            prm_t = og.params(p["t_num"], p["t_den"], p["eps"], joint=joint, strategy=strategy,
                              variant=og.OPH_VARIANT_EMPTY_AWARE)
            et = og.Results(cap)
            times, times_h = [], []
            for r_, tl in ((et, times), (er, times_h)):
                for _ in range(3):
                    r_.reset()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    og.compare_goph(qo, so, flat, prm_t if r_ is et else prm_e, r_, set_id_base=base, ws=ws[1],
                                    survivor_capacity=surv_cap)
                    e1.record()
                    torch.cuda.synchronize()
                    tl.append(e0.elapsed_time(e1))
            assert et.n() == er.n()
            variants[key] = {"ms_per_call": float(np.median(times)),
                             "ms_per_call_with_histogram": float(np.median(times_h)),
                             "mean_bins_compared": float((h * np.arange(len(h))).sum() / max(1.0, h.sum()) * kp)}
        quality["goph_empty_aware_runs"] = variants

    # ---------------- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        t0 = time.perf_counter()
        cpu_sample_step(w, CPU_SAMPLE_SETS, CPU_SAMPLE_QUERIES)
        t = time.perf_counter() - t0
        cpu = {"value": 3 * CPU_SAMPLE_QUERIES * CPU_SAMPLE_SETS / t, "unit": UNIT, "cores": oracle.num_threads(),
               "kind": "oracle",
               "sample": f"{args.config}: first {CPU_SAMPLE_SETS} sets x first {CPU_SAMPLE_QUERIES} queries, whole path "
                         f"(sketch builds incl. MinWise, 4 comparisons, threshold lists), {t:.1f} s"}

    line = {
        "metric": METRIC, "value": 3 * Q * N_total / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic",
        "config": {"workload": args.config, "sets_per_gpu": N, "sets_total": N_total, "queries": Q, "k": k,
                   "kprime": kp, "hoph_groups": L, "minwise_k": mwk, "T": f"{p['t_num']}/{p['t_den']}",
                   "epsilon": p["eps"], "parallelism": f"set-sharded x{world}",
                   "scan_strategy": ["auto", "brute", "probe"][strategy],
                   "l2": f"inputs larger than L2 (CSR {4 * nnz / 1e6:.0f} MB + sketches "
                         f"{4 * N * (k + L * hkp + mwk) / 1e9:.2f} GB per step)"},
        "value_definition": "3 * queries * sets_total / step time (each pair scored by full OPH, GOPH, HOPH)",
        "sketches_per_s": {"oph_hoph": (N_total) / (phase_ms["build_oph_hoph"] / 1e3),
                           "minwise": (N_total) / (phase_ms["build_minwise"] / 1e3)},
        "comparisons_per_s": {m: Q * N_total / (phase_ms["compare_" + m] / 1e3)
                              for m in ("full", "goph", "hoph", "minwise")},
        "phase_ms": phase_ms,
        "phase_note": "phase_ms / kernels / roofline: the K steps re-run with every call on one stream "
                      "(ms_per_step_serial); the headline ms_per_step overlaps the MinWise calls (side stream) "
                      "with the OPH family (phase_ms_concurrent)",
        "ms_per_step_serial": ms_serial,
        "phase_ms_concurrent": phase_ms_concurrent,
        "hits": hits_last,
        "roofline": roof,
        "kernels": per_kernel,
        "probe_scan": scan,
        "termination": term,
        "quality": quality,
        "device_us_per_step": {n: {"launches": v[0], "us": round(v[1], 1)} for n, v in sorted(
            kernel_us.items(), key=lambda kv: -kv[1][1])},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches * K if launches is not None else None,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="text-like", choices=CONFIG_NAMES,
                    help="workload (BASELINE.json configs); text-like is the headline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-quality", action="store_true", help="skip the precision/recall pass (untimed)")
    ap.add_argument("--no-launch-count", action="store_true", help="skip the CUPTI launch count (use under ncu)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
