"""Host-side plumbing of the sharded mode (row e) with torch.distributed gloo,
world_size 2 on CPU: trace slicing at instruction heads, the unique-id
broadcast, and the assembly of partitioned heat-map rows."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import tracegen as tg
from paper_2507_18729_b200.dist import assemble_rows, broadcast_bytes, split_at_heads


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
        # 1. the 128-byte id travels from rank 0 unchanged
        payload = bytes(range(128)) if rank == 0 else None
        got = broadcast_bytes(payload)
        # 2. partitions (disjoint chunks of 2048 cells, block-cyclic) sum to the rows
        n = 10000
        full = (np.arange(n, dtype=np.uint32) * 7919) % 1000
        own = ((np.arange(n) // 2048) % world) == rank
        part = np.where(own, full, 0).astype(np.uint32)
        rows = assemble_rows(part)
        # 3. every rank slices the same trace identically
        t = tg.random_trace(n=5000, seed=3)
        sl = split_at_heads(t.records, world)
        q.put((rank, got == bytes(range(128)), bool(np.array_equal(rows, full)), sl))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(r[1] and r[2] for r in res)
    assert res[0][3] == res[1][3]


def test_split_at_heads():
    t = tg.random_trace(n=20000, seed=4, instr_len=(1, 40))
    recs = t.records
    heads = ((recs[:, 1].to(torch.int64) >> 23) & 1).numpy()
    for P in (1, 2, 3, 7):
        sl = split_at_heads(recs, P)
        assert len(sl) == P and sl[0][0] == 0 and sl[-1][1] == recs.shape[0]
        for (a, b), (c, d) in zip(sl, sl[1:]):
            assert b == c and a <= b
        for a, b in sl[1:]:
            assert a == b or heads[a] == 1  # every non-empty slice after the first starts at a head
        sizes = [b - a for a, b in sl]
        assert max(sizes) - min(sizes) <= 2 * 40 + recs.shape[0] // P  # about even
    # degenerate inputs
    assert split_at_heads(recs[:0], 3) == [(0, 0)] * 3
    one = split_at_heads(recs[:1], 2)
    assert len(one) == 2 and sum(b - a for a, b in one) == 1 and one[0][0] == 0 and one[-1][1] == 1
