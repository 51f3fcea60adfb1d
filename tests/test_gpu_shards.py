"""Sharded mode (row e) on one GPU: nranks in-process shards
(thermo_create_local_shards, the same exchange algorithm as the NCCL ranks)
reduce slices of one trace; every job-wide output must be bit-identical to one
context reducing the same slices, and the partitions of the dense rows must be
disjoint and sum to the full rows."""
import numpy as np
import pytest

import oracle
import tracegen as tg

pytestmark = pytest.mark.gpu

WORD, SECTOR, BOTH = 1, 2, 3


def _slices(t, P):
    from paper_2507_18729_b200.dist import split_at_heads
    return [t.records[a:b] for a, b in split_at_heads(t.records, P)]


def single(t, slices, dedup, lf, ml):
    from paper_2507_18729_b200 import Thermo
    th = Thermo(max_launches=ml, max_warps_per_launch=1 << 22, dedup=dedup)
    th.register_objects(t.objects)
    for c in slices:
        if c.shape[0]:
            th.ingest(c.cuda().contiguous())
    th.build(BOTH, lf)
    return th


def sharded(t, slices, dedup, lf, ml):
    from paper_2507_18729_b200 import Thermo
    from paper_2507_18729_b200.dist import run_ranks
    shards = Thermo.local_shards(len(slices), max_launches=ml, max_warps_per_launch=1 << 22, dedup=dedup)

    def job(r):
        def f():
            th = shards[r]
            th.register_objects(t.objects)
            if slices[r].shape[0]:
                th.ingest(slices[r].cuda().contiguous())
            th.build(BOTH, lf)
        return f

    run_ranks([job(r) for r in range(len(slices))])
    return shards


def compare(t, ref, shards):
    from paper_2507_18729_b200.dist import run_ranks
    P = len(shards)
    assert [s.sharding()[:2] for s in shards] == [(r, P) for r in range(P)]
    # per-rank storage by construction (SURVEY §8e local index): rank r's dense
    # rows cover its own 2048-sector chunks only
    S_tot = sum((o[1] + 31) // 32 for o in t.objects)
    nch = (S_tot + 2047) // 2048
    for r, sh in enumerate(shards):
        own = (nch - r + P - 1) // P if nch > r else 0
        assert sh.stats()["local_sectors"] == (S_tot if P == 1 else max(1, own) * 2048)
    assert ref.stats()["local_sectors"] == S_tot
    for obj in t.objects:
        oid = obj[3]
        for gran in (WORD, SECTOR, BOTH):
            parts = [s.heatmap(oid, gran).astype(np.int64) for s in shards]
            assert np.array_equal(sum(parts), ref.heatmap(oid, gran)), (t.name, obj[4], gran)
            assert ((np.stack(parts) != 0).sum(0) <= 1).all(), "a cell is owned by two ranks"
        for gran in (WORD, SECTOR):
            for s in shards:
                assert np.array_equal(s.histogram(oid, gran), ref.histogram(oid, gran)), (t.name, obj[4], gran)
    rpc = ref.per_pc(WORD), ref.per_pc(SECTOR)
    for s in shards:
        for gran, rows in zip((WORD, SECTOR), rpc):
            got = s.per_pc(gran)
            assert [(a, b) for a, b, _ in got] == [(a, b) for a, b, _ in rows]
            for (_, _, h1), (_, _, h2) in zip(got, rows):
                assert np.array_equal(h1, h2)
    ri = ref.classify()
    for got in run_ranks([s.classify for s in shards]):
        assert got == ri, t.name
    rs = ref.stats()
    for s in shards:
        st = s.stats()
        for f in ("records", "invalid", "unmapped_words", "mapped_word_accesses", "distinct_pairs", "n_pcs"):
            assert st[f] == rs[f], (t.name, f, st[f], rs[f])


CASES = [
    lambda: tg.gemm(256, 256, 64, "v00"),
    lambda: tg.stencil(256),
    lambda: tg.random_trace(n=40000, seed=5, n_warps=200, n_launches=3, max_len=300000),
    lambda: tg.synthetic(n_objects=16, n_launches=2, warps_per_launch=64, records_per_warp=256, size_shift=12),
]


def _one_sector():
    # one 32-byte sector read by 60 k warps (a multi-pass big sector on its owner
    # rank, the other ranks' keys reaching it through the exchange)
    from tests.test_gpu_parity import _one_sector_trace
    return _one_sector_trace()


CASES.append(_one_sector)


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("dedup", [1, 2, 3])
@pytest.mark.parametrize("i", range(len(CASES)))
def test_shards_match_one_context(i, dedup, P):
    t = CASES[i]()
    ml = max(1, int(t.meta.get("launches", 1)))
    sl = _slices(t, P)
    ref = single(t, sl, dedup, oracle.ALL_LAUNCHES, ml)
    compare(t, ref, sharded(t, sl, dedup, oracle.ALL_LAUNCHES, ml))


def test_shards_launch_filter_rebuild_and_late_ingest():
    from paper_2507_18729_b200.dist import run_ranks
    t = tg.random_trace(n=30000, seed=9, n_warps=100, n_launches=3, max_len=300000)
    P, ml = 3, 3
    sl = _slices(t, P)
    # each slice in two ingest calls, the second starting at an instruction head
    from paper_2507_18729_b200.dist import split_at_heads
    first, late = [], []
    for s in sl:
        (a, b), (c, d) = split_at_heads(s, 2)
        first.append(s[a:b])
        late.append(s[c:d])
    shards = sharded(t, first, 0, oracle.ALL_LAUNCHES, ml)
    ref = single(t, first, 0, oracle.ALL_LAUNCHES, ml)
    compare(t, ref, shards)
    # rebuild with each launch filter from the retained (exchanged) keys
    for lf in range(ml):
        run_ranks([lambda s=s: s.build(BOTH, lf) for s in shards])
        ref.build(BOTH, lf)
        compare(t, ref, shards)

    # ingest more after a build, build again (only the new keys move)
    def more(r):
        def f():
            if late[r].shape[0]:
                shards[r].ingest(late[r].cuda().contiguous())
            shards[r].build(BOTH, oracle.ALL_LAUNCHES)
        return f

    run_ranks([more(r) for r in range(P)])
    for c in late:
        if c.shape[0]:
            ref.ingest(c.cuda().contiguous())
    ref.build(BOTH, oracle.ALL_LAUNCHES)
    compare(t, ref, shards)


def test_shards_empty_rank():
    """More ranks than instruction heads: some ranks hold no records."""
    t = tg.tiny("B")
    sl = [t.records, t.records[:0], t.records[:0], t.records[:0]]
    ref = single(t, [t.records], 0, oracle.ALL_LAUNCHES, 1)
    compare(t, ref, sharded(t, sl, 0, oracle.ALL_LAUNCHES, 1))


def test_nccl_transport_single_rank(monkeypatch):
    """The NCCL transport (thermo_create_dist) with one rank, forced on: init,
    all-reduce, all-gather and the all-to-all's self copy through NCCL on one
    GPU, against a plain context."""
    monkeypatch.setenv("THERMO_FORCE_COMM", "1")
    from paper_2507_18729_b200 import Thermo
    from paper_2507_18729_b200.thermo import nccl_unique_id
    t = tg.random_trace(n=30000, seed=11, n_warps=100, n_launches=2, max_len=300000)
    th = Thermo.dist(nccl_unique_id(), 0, 1, max_launches=2, max_warps_per_launch=1 << 22)
    th.register_objects(t.objects)
    th.ingest(t.records.cuda().contiguous())
    th.build(BOTH, oracle.ALL_LAUNCHES)
    ref = single(t, [t.records], 0, oracle.ALL_LAUNCHES, 2)
    compare(t, ref, [th])


def test_shards_warp_records():
    """Warp-instruction records (f4) ingested by 3 in-process shards: same
    job-wide result as one context."""
    from paper_2507_18729_b200 import Thermo
    from paper_2507_18729_b200.dist import run_ranks
    objects, recs = tg.random_warp_trace(n_instr=6000, seed=21, n_launches=2, max_len=300000)
    t = tg.Trace("warp-shards", objects, recs, meta=dict(launches=2))
    parts = [recs[i::3].contiguous() for i in range(3)]  # any split: every warp record is one instruction
    ref = Thermo(max_launches=2, max_warps_per_launch=1 << 22)
    ref.register_objects(objects)
    for p in parts:
        ref.ingest_warp(p.cuda())
    ref.build(BOTH)
    shards = Thermo.local_shards(3, max_launches=2, max_warps_per_launch=1 << 22)

    def job(r):
        def f():
            shards[r].register_objects(objects)
            shards[r].ingest_warp(parts[r].cuda())
            shards[r].build(BOTH)
        return f

    run_ranks([job(r) for r in range(3)])
    compare(t, ref, shards)


@pytest.mark.parametrize("P", [2, 3])
def test_shards_dense_block_mode_and_whitelist(P):
    """Row e with SURVEY §8f item 1: sampled-block mode (AUTO = DENSE warp
    bitmasks) plus a launch whitelist, sharded over P in-process ranks, equals
    one context on the same slices."""
    from paper_2507_18729_b200 import Thermo
    from paper_2507_18729_b200.dist import run_ranks
    t = tg.synthetic(n_objects=16, n_launches=4, warps_per_launch=256, records_per_warp=256, size_shift=12)
    cfg = dict(max_launches=4, max_warps_per_launch=1 << 22, block_warps=64, block_id=1)
    sl = _slices(t, P)
    ref = Thermo(**cfg)
    ref.register_objects(t.objects)
    ref.set_launch_whitelist([0, 2, 3])
    for c in sl:
        if c.shape[0]:
            ref.ingest(c.cuda().contiguous())
    ref.build(BOTH)
    assert ref.stats()["dedup_used"] == 4
    shards = Thermo.local_shards(P, **cfg)

    def job(r):
        def f():
            th = shards[r]
            th.register_objects(t.objects)
            th.set_launch_whitelist([0, 2, 3])
            if sl[r].shape[0]:
                th.ingest(sl[r].cuda().contiguous())
            th.build(BOTH)
        return f

    run_ranks([job(r) for r in range(P)])
    assert all(s.stats()["dedup_used"] == 4 for s in shards)
    compare(t, ref, shards)
