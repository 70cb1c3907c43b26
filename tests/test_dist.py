"""Multi-process (world_size 2, gloo, CPU) tests of the sharding / gather
plumbing used by bench.py's N>1 path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_11254_b200 import HIT_DTYPE
from paper_1805_11254_b200 import dist as odist


def test_shard_range_covers_exactly():
    for n in (0, 1, 7, 200_000, 10_000_001):
        for world in (1, 2, 3, 8):
            rs = [odist.shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [hi - lo for lo, hi in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        odist.shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r holds r+2 records (rank 1 holds a padded buffer larger than its count)
        n = rank + 2
        rec = np.zeros(8, dtype=HIT_DTYPE)
        rec["query"][:n] = np.arange(n) + 10 * rank
        rec["set_id"][:n] = 1000 * rank + np.arange(n)
        rec["estimate"][:n] = 0.5
        u8 = torch.from_numpy(rec.view(np.uint8).copy())
        allh, counts = odist.gather_hits(u8, n)
        got = odist.records_from_bytes(allh)
        # query broadcast from rank 0
        t = torch.arange(5, dtype=torch.int32) if rank == 0 else torch.zeros(5, dtype=torch.int32)
        odist.broadcast_tensors([t])
        mx = odist.max_over_ranks(float(rank + 1))
        q.put((rank, counts, got["set_id"].tolist(), got["query"].tolist(), t.tolist(), mx))
    finally:
        dist.destroy_process_group()


def test_gather_hits_and_broadcast_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, counts, sids, qs, t, mx in out:
        assert counts == [2, 3]
        assert sids == [0, 1, 1000, 1001, 1002]
        assert qs == [0, 1, 10, 11, 12]
        assert t == [0, 1, 2, 3, 4]
        assert mx == 2.0


def _records_from_oracle(recs, set_id_base):
    """oph_hit records of the Similar pairs of an oracle result matrix (the records a
    rank's compare call appends), in arbitrary (here: reversed) order."""
    q, s = np.nonzero(recs["verdict"] == 1)
    out = np.zeros(len(q), dtype=HIT_DTYPE)
    out["query"], out["set_id"] = q, s + set_id_base
    out["n_mb"], out["n_excl"] = recs["n_mb"][q, s], recs["n_excl"][q, s]
    out["groups"], out["verdict"], out["flags"] = recs["groups"][q, s], 1, recs["flags"][q, s]
    out["estimate"] = recs["estimate"][q, s]
    return out[::-1].copy()


def _shard_worker(rank, world, port, q):
    """The N > 1 step of bench.py with the CPU oracle standing in for the compare kernels:
    rank r scores its contiguous shard of the tiny collection with set IDs offset by its
    shard base, the hit records are gathered (gather_hits) and rank 0 merges them."""
    import oracle
    from workloads import tiny
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = tiny()
        p = w.params
        lo, hi = odist.shard_range(w.n_sets, rank, world)
        sh = w.slice_sets(lo, hi)
        F = oracle.oph_sketch(sh.offsets, sh.ids, w.vocab_size, p["k"], p["perm_seed"])
        QF = oracle.oph_sketch(w.q_offsets, w.q_ids, w.vocab_size, p["k"], p["perm_seed"])
        out = {}
        for m in ("full", "goph"):
            if m == "full":
                r = oracle.compare_full(QF, F, t_num=p["t_num"], t_den=p["t_den"], groups=p["k"] // p["kprime"])
            else:
                r = oracle.compare_goph(QF, F, n=p["k"] // p["kprime"], kprime=p["kprime"], t_num=p["t_num"],
                                        t_den=p["t_den"], eps=p["eps"])
            rec = _records_from_oracle(r, lo)
            buf = torch.zeros(max(1, len(rec)) * 20 + 40, dtype=torch.uint8)
            buf[: len(rec) * 20] = torch.from_numpy(rec.view(np.uint8).copy())
            allh, counts = odist.gather_hits(buf, len(rec))
            merged = odist.merge_threshold_records(odist.records_from_bytes(allh))
            out[m] = (counts, merged.tobytes())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_sharded_compare_gather_merge_gloo():
    """shards with set_id_base offsets -> per-shard records -> gather -> merge
    on rank 0 == the unsharded threshold list with the unsharded records, byte for byte."""
    import oracle
    from workloads import tiny
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = tiny()
    p = w.params
    F = oracle.oph_sketch(w.offsets, w.ids, w.vocab_size, p["k"], p["perm_seed"])
    QF = oracle.oph_sketch(w.q_offsets, w.q_ids, w.vocab_size, p["k"], p["perm_seed"])
    want = {"full": oracle.compare_full(QF, F, t_num=p["t_num"], t_den=p["t_den"], groups=p["k"] // p["kprime"]),
            "goph": oracle.compare_goph(QF, F, n=p["k"] // p["kprime"], kprime=p["kprime"], t_num=p["t_num"],
                                        t_den=p["t_den"], eps=p["eps"])}
    for m, recs in want.items():
        full = odist.merge_threshold_records(_records_from_oracle(recs, 0))
        assert len(full) > 0
        for rank in range(world):
            counts, merged = out[rank][m]
            assert sum(counts) == len(full)
            assert merged == full.tobytes(), (m, rank)
        assert [(int(a), int(b)) for a, b in zip(full["query"], full["set_id"])] == oracle.threshold_list(recs)


def test_bench_refuses_world_size_mismatch():
    """bench.py --gpus N must match the launcher's WORLD_SIZE (no silent 1-rank run)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "1"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr
