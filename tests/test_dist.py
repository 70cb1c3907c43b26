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
