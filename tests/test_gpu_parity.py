"""GPU parity: libthermo (through its C ABI) against the CPU oracle, element by
element, bit-exact (all outputs are integers; BJ north_star "must match the
oracle bit-exactly").  Sizes span several decode ranges / sort tiles with
ragged tails; full-size configs are checked on sampled sectors and closed forms.
"""
import numpy as np
import pytest
import torch

import oracle
import tracegen as tg

pytestmark = pytest.mark.gpu

WORD, SECTOR, BOTH = 1, 2, 3


def gpu_ctx(t, dedup=0, max_launches=None, track_pc=True):
    from paper_2507_18729_b200 import Thermo
    ml = max_launches or max(1, int(t.meta.get("launches", 1)))
    th = Thermo(max_launches=ml, max_warps_per_launch=1 << 22, max_pcs=4096, dedup=dedup, track_pc=track_pc)
    th.register_objects(t.objects)
    return th


def run_both(t, calls=None, dedup=0, launch_filter=oracle.ALL_LAUNCHES, max_launches=None, host=False):
    calls = calls if calls is not None else t.calls()
    orc = oracle.run([o[:4] for o in t.objects], calls, launch_filter)
    th = gpu_ctx(t, dedup, max_launches)
    for c in calls:
        th.ingest(c.contiguous() if host else c.cuda().contiguous())
    th.build(BOTH, launch_filter)
    return orc, th


def compare(orc, th, t, check_pc=True, check_ind=True):
    for k, obj in enumerate(t.objects):
        oid = obj[3]
        w, s = th.heatmap(oid, WORD), th.heatmap(oid, SECTOR)
        ow, os_ = orc.word_counts(k), orc.sector_counts(k)
        assert np.array_equal(w, ow), (t.name, obj[4], "word", np.nonzero(w != ow)[0][:10])
        assert np.array_equal(s, os_), (t.name, obj[4], "sector", np.nonzero(s != os_)[0][:10])
        assert np.array_equal(th.histogram(oid, WORD), orc.hist(k, False)), (t.name, obj[4])
        assert np.array_equal(th.histogram(oid, SECTOR), orc.hist(k, True)), (t.name, obj[4])
        both = th.heatmap(oid, BOTH).reshape(-1, 9)
        assert np.array_equal(both[:, 8], os_)
    if check_pc:
        rows = orc.per_pc()
        gw, gs = th.per_pc(WORD), th.per_pc(SECTOR)
        assert [(r[0], r[1]) for r in rows] == [(r[0], r[1]) for r in gw] == [(r[0], r[1]) for r in gs]
        for r, a, b in zip(rows, gw, gs):
            assert np.array_equal(r[2], a[2]), (t.name, hex(r[1]))
            assert np.array_equal(r[3], b[2]), (t.name, hex(r[1]))
    if check_ind:
        oi, gi = orc.classify(), th.classify()
        for k, (a, b) in enumerate(zip(oi, gi)):
            for f, v in a.items():
                assert b[f] == v, (t.name, t.objects[k][4], f, v, b[f])
    st, ost = th.stats(), orc.stats()
    for f in ("records", "invalid", "unmapped_words", "mapped_word_accesses"):
        assert st[f] == ost[f], (f, st[f], ost[f])


SMALL = [
    lambda: tg.tiny("A"), lambda: tg.tiny("B"), lambda: tg.fig3("a"), lambda: tg.fig3("b"),
    lambda: tg.fig6(3, 16), lambda: tg.fig6(8, 0), lambda: tg.gemm(64, 64, 16, "v00"),
    lambda: tg.gemm(128, 96, 40, "v01"), lambda: tg.stencil(96), lambda: tg.spmv(10, 8),
    lambda: tg.strided_gather(64, 1024, 3), lambda: tg.smem_thread_local(), lambda: tg.smem_warp_broadcast(),
]


@pytest.mark.parametrize("dedup", [1, 2, 3])
@pytest.mark.parametrize("i", range(len(SMALL)))
def test_small_workloads(i, dedup):
    t = SMALL[i]()
    orc, th = run_both(t, dedup=dedup)
    compare(orc, th, t)


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("dedup", [1, 2, 3])
def test_random_traces(seed, dedup):
    """Unaligned/straddling sizes, unmapped and invalid records, 3 launches,
    shared-space objects, instructions of 1..40 records (split at 32)."""
    t = tg.random_trace(n=30000 + 777 * seed, seed=seed, n_warps=300, n_launches=3)
    t.meta["launches"] = 3
    calls = [t.records[a:b] for a, b in tg.split_calls(t.n, t.records, 3)]
    for lf in (oracle.ALL_LAUNCHES, 2):
        orc, th = run_both(t, calls=calls, dedup=dedup, launch_filter=lf)
        compare(orc, th, t)


def _gap_trace(pattern, n_words, reps):
    """One warp reads words w of a 4-byte array whenever pattern[w % len] is
    set, 32 lanes per instruction: the touched words' gaps repeat the
    pattern's (e.g. 1, 2, 1, 2 ...)."""
    objects = [(0x500000, 4 * n_words, 0, 0, "gaps")]
    words = [w for w in range(n_words) if pattern[w % len(pattern)]][:reps]
    n = (len(words) + 31) // 32 * 32
    addr = torch.tensor(words + [words[-1]] * (n - len(words)), dtype=torch.int64).reshape(-1, 32) * 4 + 0x500000
    act = torch.arange(n).reshape(-1, 32) < len(words)
    rec = tg.from_instructions(addr, act, 0, 0x700, 0, 2)
    return tg.Trace("gaps", objects, rec, meta=dict(warps=1, launches=1))


@pytest.mark.parametrize("pattern,reps", [((1, 1, 0), 20001), ((1, 1, 0), 20000), ((1, 0, 1, 1, 0, 0), 30001),
                                          ((1,) * 7 + (0,), 50000), ((1, 0, 0), 40000)])
def test_dominant_gap_majority_boundary(pattern, reps):
    """The dominant gap needs a strict majority of the gaps: gaps 1, 2
    alternating (1 holds exactly half, or one more than half), a gap of 1 in
    3 of 5, gaps of 1 in 6 of 7 (the first pass's exact count of 1-gaps), and
    all gaps 3 (the verify scan) -- against the oracle on every indicator field."""
    t = _gap_trace(pattern, 3 * reps, reps)
    orc, th = run_both(t)
    compare(orc, th, t)


@pytest.mark.parametrize("n_pcs", [8, 9])
def test_random_traces_pc_count_boundary(n_pcs):
    """SEGMENT's per-pc path switches at 8 pc ids in the job (byte masks and a
    direct bin table up to 8, a second hash set above): both sides, with a
    launch-filtered rebuild."""
    t = tg.random_trace(n=40000, seed=11 + n_pcs, n_warps=400, n_launches=1, n_pcs=n_pcs)
    t.meta["launches"] = 1
    for lf in (oracle.ALL_LAUNCHES, 0):
        orc, th = run_both(t, dedup=3, launch_filter=lf)
        compare(orc, th, t)
        assert th.stats()["n_pcs"] == n_pcs


@pytest.mark.parametrize("dist", ["bimodal", "uniform"])
@pytest.mark.parametrize("dedup", [1, 2, 3])
def test_random_hot(dist, dedup):
    """RandomHot (Fig. 5(f)): 8192 sectors = 4 indicator
    tiles, ~1.05 M records, word temps 3/29 (bimodal: CV 0.81 -> RandomHot) or
    3..29 (uniform: CV 0.487 -> Hot) drawn per word.  Every output bit-exact
    against the oracle, and the label itself asserted."""
    T = tg.hot_temps(8192, dist)
    t = tg.hot_spots(T)
    assert t.n >= 10 ** 5
    orc, th = run_both(t, dedup=dedup)
    compare(orc, th, t)
    want = "RandomHot" if dist == "bimodal" else "Hot"
    assert oracle.label_names(th.classify()[0]["labels"]) == [want]
    # shuffled instructions in 3 ingest calls: the same result
    sh = tg.shuffle_instructions(t.records, 5)
    calls = [sh[a:b] for a, b in tg.split_calls(t.n, sh, 3)]
    orc2, th2 = run_both(t, calls=calls, dedup=dedup)
    compare(orc2, th2, t)


@pytest.mark.parametrize("lo,hi,want", [(16, 48, "Hot"), (16, 49, "RandomHot")])
def test_random_hot_cv_boundary(lo, hi, want):
    """Population CV exactly 1/2 (16/48) is not 'exceeds': Hot; 16/49: RandomHot."""
    t = tg.hot_spots(torch.tensor([lo, hi] * (4 * 2048)))
    orc, th = run_both(t)
    compare(orc, th, t)
    assert oracle.label_names(th.classify()[0]["labels"]) == [want]


@pytest.mark.parametrize("decoder", ["view", "lane"])
@pytest.mark.parametrize("make", [lambda: tg.random_trace(n=30000, seed=31, n_warps=300, n_launches=3),
                                  lambda: tg.spmv(11, 8), lambda: tg.gemm(64, 64, 16, "v00"),
                                  lambda: tg.stencil(96), lambda: tg.hot_spots(tg.hot_temps(2048, "bimodal"))])
def test_both_decoders(decoder, make, monkeypatch):
    """Both per-lane decoders (the view-per-instruction kernel and the
    lane-per-record kernel; AUTO picks one by the mean instruction length)
    forced on the same traces, every output against the oracle."""
    monkeypatch.setenv("THERMO_DECODER", decoder)
    t = make()
    t.meta.setdefault("launches", 3)
    calls = [t.records[a:b] for a, b in tg.split_calls(t.n, t.records, 3)]
    orc, th = run_both(t, calls=calls)
    compare(orc, th, t)


def test_launch_filter_rebuild_and_host_ingest():
    t = tg.random_trace(n=20000, seed=21, n_launches=4)
    t.meta["launches"] = 4
    orc, th = run_both(t, host=True)       # host-pointer ingest (staged by the library)
    compare(orc, th, t)
    for lf in range(4):                     # build again from the retained keys
        th.build(BOTH, lf)
        o2 = oracle.run([o[:4] for o in t.objects], t.calls(), lf)
        compare(o2, th, t)


def test_permutation_and_duplication_invariance():
    t = tg.gemm(64, 64, 24, "v00")
    perm = tg.shuffle_instructions(t.records, 7)
    dup = torch.cat([t.records, perm])
    ref = None
    for calls in ([t.records], [perm], [dup], [t.records[a:b] for a, b in tg.split_calls(t.n, t.records, 6)]):
        th = gpu_ctx(t)
        for c in calls:
            th.ingest(c.cuda().contiguous())
        th.build()
        out = [th.heatmap(o[3], BOTH) for o in t.objects]
        if ref is None:
            ref = out
        for a, b in zip(ref, out):
            assert np.array_equal(a, b)


def test_empty_and_degenerate():
    from paper_2507_18729_b200 import Thermo, ThermoError
    t = tg.tiny("B")
    th = gpu_ctx(t)
    th.ingest(t.records[:0].cuda())        # empty call is a no-op
    with pytest.raises(ThermoError):        # nothing ingested yet
        th.build()
    th.ingest(t.records[:1].cuda())         # a single record
    th.build()
    w = th.heatmap(0, WORD)
    assert w[0] == 1 and w.sum() == 1
    with pytest.raises(ThermoError):
        th.register_objects(t.objects)      # second registration
    th2 = Thermo()
    with pytest.raises(ThermoError):
        th2.register_objects([(0x1010, 64, 0, 0)])  # misaligned base
    th3 = Thermo()
    with pytest.raises(ThermoError):
        th3.register_objects([(0x1000, 64, 0, 0), (0x1020, 64, 0, 1)])  # overlap
    # out-of-range warp id -> ERANGE at build
    th4 = Thermo(max_warps_per_launch=4)
    th4.register_objects(t.objects)
    th4.ingest(t.records.cuda())
    with pytest.raises(ThermoError):
        th4.build()


def test_gemm_full_size_all_outputs():
    """BJ configs[1] at full size (270,532,608 records) in the bench's launch
    configuration: closed forms on every cell, then the UNRESTRICTED oracle over
    all records compared on every output -- every dense word and sector row,
    both histograms of every object, every per-PC row, every indicator field and
    label, and the stats counters."""
    t = tg.gemm(1024, 1024, 128, "v00", device="cuda")
    th = gpu_ctx(t)
    th.ingest(t.records)
    th.build()
    wa, sa = th.heatmap(0, WORD), th.heatmap(0, SECTOR)
    assert (wa == 1024).all() and (sa == 1024).all()
    assert (th.heatmap(1, WORD) == 32).all() and (th.heatmap(1, SECTOR) == 256).all()
    assert (th.heatmap(2, WORD) == 1).all() and (th.heatmap(2, SECTOR) == 8).all()
    labels = [oracle.label_names(r["labels"]) for r in th.classify()]
    assert labels == [["Hot"], ["FalseSharing"], ["FalseSharing"]]
    st = th.stats()
    assert st["records"] == 270532608 and st["distinct_pairs"] == 22020096
    recs = t.records.cpu()
    t.records = recs
    orc = oracle.Oracle([o[:4] for o in t.objects])
    for a in range(0, recs.shape[0], 1 << 25):
        orc.ingest(recs[a:a + (1 << 25)])
    orc.build()
    compare(orc, th, t)


def test_stencil_full_size_closed_form_all_cells():
    """BJ configs[2] at full size (8192^2 column-mapped 5-point stencil,
    402,456,600 records): every word and sector of `in` and `out`, both
    histograms of both objects, every per-PC row and the distinct-pair totals
    against the reader enumeration of tests/closed_forms.py (pinned to the
    oracle at N = 64, 96, 128 in test_oracle_pins.py).  Distinct (sector, warp)
    pairs in closed form: `in` has sum over row blocks |R| (cols + cols with
    j % 8 in {0, 7}) + 2 * 256 * 8190 = 8190 * 10236 + 4,193,280 = 88,026,120,
    `out` 8190^2 = 67,076,100, total 155,102,220; distinct (pc, sector) pairs
    50,319,360."""
    from tests import closed_forms as C
    N = 8192
    t = tg.stencil(N, device="cuda")
    assert t.n == 6 * (N - 2) ** 2
    from paper_2507_18729_b200 import Thermo
    th = Thermo(max_launches=1, max_warps_per_launch=1 << 21, max_pcs=64)
    th.register_objects(t.objects)
    th.ingest(t.records)
    th.build()
    del t
    torch.cuda.empty_cache()
    st = th.stats()
    assert st["distinct_pairs"] == 8190 * 10236 + 4_193_280 + 8190 ** 2 == 155_102_220
    assert st["distinct_pc_pairs"] == 50_319_360
    assert st["records"] == 402_456_600 and st["invalid"] == 0 and st["unmapped_words"] == 0
    w_in, s_in, w_out, s_out = C.stencil_counts(N, device="cuda")
    exp = ((w_in, s_in), (w_out, s_out))
    for k, (wc, sc) in enumerate(exp):
        assert np.array_equal(th.heatmap(k, WORD), wc.cpu().numpy().reshape(-1).astype(np.uint32)), k
        assert np.array_equal(th.heatmap(k, SECTOR), sc.cpu().numpy().reshape(-1).astype(np.uint32)), k
        assert np.array_equal(th.histogram(k, WORD), C.level_hist(wc).cpu().numpy()), k
        assert np.array_equal(th.histogram(k, SECTOR), C.level_hist(sc).cpu().numpy()), k
    assert int(s_in.sum()) + int(s_out.sum()) == st["distinct_pairs"]
    gw, gs = th.per_pc(WORD), th.per_pc(SECTOR)
    assert [r[1] for r in gw] == list(C.STENCIL_PCS) == [r[1] for r in gs]
    npc = 0
    for k in range(6):
        wm, sm = C.stencil_pc_cells(N, k, device="cuda")
        wc, sc = exp[0] if k < 5 else exp[1]
        assert np.array_equal(gw[k][2], C.level_hist(wc[wm]).cpu().numpy()), hex(C.STENCIL_PCS[k])
        assert np.array_equal(gs[k][2], C.level_hist(sc[sm]).cpu().numpy()), hex(C.STENCIL_PCS[k])
        npc += int(sm.sum())
    assert npc == st["distinct_pc_pairs"]
    ind = th.classify()
    for k, (wc, sc) in enumerate(exp):
        assert ind[k]["touched_sectors"] == int((sc > 0).sum()) and ind[k]["touched_words"] == int((wc > 0).sum())
        assert ind[k]["sum_x"] == int(wc.to(torch.int64).sum()) and ind[k]["max_sector_count"] == int(sc.max())
        assert ind[k]["sum_x2_lo"] + (ind[k]["sum_x2_hi"] << 64) == int((wc.to(torch.int64) ** 2).sum())
    assert oracle.label_names(ind[1]["labels"]) == ["FalseSharing"]


def _hot_sector_trace(n=40000, hot_warps=6000, seed=3):
    """A hot object (2 sectors read by thousands of warps, more keys than a
    SEGMENT chunk holds) beside a spread one; instructions of 1-3 records
    (packed into multi-instruction views by the fast decoder)."""
    import torch
    g = torch.Generator().manual_seed(seed)
    objects = [(0x100000, 64, 0, 7, "hot"), (0x200000, 1 << 16, 0, 8, "spread")]
    hot = torch.rand(n, generator=g) < 0.5
    addr = torch.where(hot, 0x100000 + 4 * torch.randint(0, 16, (n,), generator=g),
                       0x200000 + 4 * torch.randint(0, 1 << 14, (n,), generator=g))
    warp = torch.where(hot, torch.randint(0, hot_warps, (n,), generator=g), torch.randint(0, 100, (n,), generator=g))
    # instructions: a record starts one with probability 1/2 and then shares the warp/pc of its head
    istart = (torch.rand(n, generator=g) < 0.5).to(torch.int64)
    istart[0] = 1
    iid = torch.cumsum(istart, 0) - 1
    heads = torch.nonzero(istart).flatten()
    warp = warp[heads][iid]
    hot = hot[heads][iid]
    addr = torch.where(hot, 0x100000 + (addr & 63), 0x200000 + (addr & 0xFFFF))
    pc = torch.where(hot, 0x500, 0x510 + 16 * (iid % 3))
    rec = tg.pack_records(addr, 2, 0, 0, istart, warp, pc, 0)
    return tg.Trace("hot-sector", objects, rec, meta=dict(warps=hot_warps, launches=1))


@pytest.mark.parametrize("dedup", [0, 1, 2, 3])
def test_hot_sector_and_short_instructions(dedup):
    t = _hot_sector_trace()
    orc, th = run_both(t, dedup=dedup)
    compare(orc, th, t)
    if dedup in (0, 3):
        assert th.stats()["dedup_used"] == 3  # SEGMENT with its big-sector side path, no fallback


def _one_sector_trace(n_warps=60000):
    """Every warp loads the 8 words of a 32-byte counter block (one sector) and
    one word of a 256-byte array: 9 registered sectors for 120 k keys, far
    below keys / 2048 (the SEGMENT chunk tables are sized by sectors)."""
    objects = [(0x300000, 32, 0, 0, "counter"), (0x400000, 256, 0, 1, "arr")]
    w = torch.arange(n_warps, dtype=torch.int64)
    lane = torch.arange(32, dtype=torch.int64)
    a0 = (0x300000 + 4 * (lane % 8)).unsqueeze(0).expand(n_warps, 32)
    a1 = (0x400000 + 4 * ((w % 64).unsqueeze(1) + 0 * lane)).expand(n_warps, 32)
    act0 = (lane < 8).unsqueeze(0).expand(n_warps, 32)
    act1 = (lane == 0).unsqueeze(0).expand(n_warps, 32)
    addr = torch.stack([a0, a1], 1).reshape(-1, 32)
    act = torch.stack([act0, act1], 1).reshape(-1, 32)
    wid = w.repeat_interleave(2)
    pc = torch.tensor([0x600, 0x610], dtype=torch.int64).repeat(n_warps)
    rec = tg.from_instructions(addr, act, wid, pc, 0, 2)
    return tg.Trace("one-sector", objects, rec, meta=dict(warps=n_warps, launches=1))


@pytest.mark.parametrize("dedup", [0, 1, 2])
def test_one_hot_sector_many_warps(dedup):
    t = _one_sector_trace()
    orc, th = run_both(t, dedup=dedup)
    compare(orc, th, t)
    assert th.heatmap(0, SECTOR).tolist() == [60000]
    assert th.heatmap(0, WORD).tolist() == [60000] * 8


@pytest.mark.parametrize("case", ["tiny", "fig3a", "fig3b", "gemm", "stencil", "random", "hot"])
def test_access_counts(case):
    """Access counts: lane accesses per word, every
    launch, through thermo_query_access, against the oracle."""
    from paper_2507_18729_b200 import Thermo
    t = {"tiny": lambda: tg.tiny("B"), "fig3a": lambda: tg.fig3("a"), "fig3b": lambda: tg.fig3("b"),
         "gemm": lambda: tg.gemm(128, 96, 40, "v01"), "stencil": lambda: tg.stencil(96),
         "random": lambda: tg.random_trace(n=30000, seed=8, n_warps=300, n_launches=3),
         "hot": lambda: _hot_sector_trace()}[case]()
    ml = max(1, int(t.meta.get("launches", 1)))
    th = Thermo(max_launches=ml, max_warps_per_launch=1 << 22, track_access=True)
    th.register_objects(t.objects)
    calls = t.calls() if case != "random" else [t.records[a:b] for a, b in tg.split_calls(t.n, t.records, 3)]
    for c in calls:
        th.ingest(c.cuda().contiguous())
    orc = oracle.run([o[:4] for o in t.objects], calls, 1 if case == "random" else oracle.ALL_LAUNCHES)
    for k, obj in enumerate(t.objects):
        assert np.array_equal(th.access(obj[3]), orc.access_counts(k)), (case, obj[4])
    th.build(BOTH)  # the heat map is unaffected by track_access
    orc2 = oracle.run([o[:4] for o in t.objects], calls)
    for k, obj in enumerate(t.objects):
        assert np.array_equal(th.heatmap(obj[3], WORD), orc2.word_counts(k))


@pytest.mark.parametrize("dedup", [0, 3, 4])  # AUTO (= DENSE here), SEGMENT, DENSE
@pytest.mark.parametrize("block", [0, 5])
def test_sampled_block_mode(block, dedup):
    """Sampled-block mode: only one thread
    block's warps are reduced; everything against the oracle's block scope,
    on a fuzz trace (mixed/invalid records, general path) and on SGEMM, with
    the DENSE warp-bitmask path and with SEGMENT."""
    from paper_2507_18729_b200 import Thermo
    for t, bw in ((tg.gemm(128, 96, 40, "v00"), 32),
                  (tg.random_trace(n=30000, seed=13, n_warps=400, n_launches=1), 16)):
        th = Thermo(max_launches=1, max_warps_per_launch=1 << 22, block_warps=bw, block_id=block, dedup=dedup)
        th.register_objects(t.objects)
        th.ingest(t.records.cuda().contiguous())
        th.build(BOTH)
        orc = oracle.Oracle([o[:4] for o in t.objects])
        orc.block_scope(bw, block)
        orc.ingest(t.records)
        orc.build()
        compare(orc, th, t)
        assert th.stats()["dedup_used"] == (4 if dedup in (0, 4) else dedup)


@pytest.mark.parametrize("bw,block", [(64, 2), (8, 31)])
def test_dense_multi_launch(bw, block):
    """DENSE on the synthetic generator's 8 launches x 256
    warps: one block of 64 (or 8) warps per launch; every output against the
    oracle's block scope, for all launches and for one launch (G2)."""
    from paper_2507_18729_b200 import Thermo
    t = tg.synthetic(n_objects=16, n_launches=8, warps_per_launch=256, records_per_warp=256, size_shift=14)
    th = Thermo(max_launches=8, max_warps_per_launch=256, max_pcs=64, block_warps=bw, block_id=block,
                dedup=4)
    th.register_objects(t.objects)
    th.ingest(t.records.cuda())
    for lf in (None, 5):
        th.build(BOTH) if lf is None else th.build(BOTH, lf)
        orc = oracle.Oracle([o[:4] for o in t.objects])
        orc.block_scope(bw, block)
        for c in t.calls():
            orc.ingest(c)
        orc.build() if lf is None else orc.build(lf)
        compare(orc, th, t)
        assert th.stats()["dedup_used"] == 4


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("dedup", [0, 1, 2])
def test_warp_records_random(seed, dedup):
    """Warp-instruction records through
    thermo_ingest_warp_trace against the oracle's ingest_warp: random active
    masks, unaligned/straddling sizes, lanes outside objects, invalid flags and
    address bits >= 48 (spilled to the per-lane kernels), 2 launches."""
    from paper_2507_18729_b200 import Thermo
    objects, recs = tg.random_warp_trace(n_instr=4000 + 300 * seed, seed=seed, n_launches=2, max_len=20000)
    t = tg.Trace("warp-random", objects, recs, meta=dict(launches=2))
    th = Thermo(max_launches=2, max_warps_per_launch=1 << 22, dedup=dedup, track_access=True)
    th.register_objects(objects)
    half = recs.shape[0] // 2
    th.ingest_warp(recs[:half].cuda().contiguous())
    th.ingest_warp(recs[half:].contiguous())  # host pointer
    th.build(BOTH)
    orc = oracle.Oracle([o[:4] for o in objects])
    orc.ingest_warp(recs[:half])
    orc.ingest_warp(recs[half:])
    orc.build()
    compare(orc, th, t)
    for k, o in enumerate(objects):
        assert np.array_equal(th.access(o[3]), orc.access_counts(k))


@pytest.mark.parametrize("make", [lambda: tg.tiny("B"), lambda: tg.gemm(128, 96, 40, "v00"), lambda: tg.stencil(96),
                                  lambda: tg.spmv(10, 8)])
def test_warp_records_workloads(make):
    t = make()
    w = tg.to_warp_records(t.records)
    from paper_2507_18729_b200 import Thermo
    th = gpu_ctx(t)
    th.ingest_warp(w.cuda())
    th.build(BOTH)
    orc = oracle.run([o[:4] for o in t.objects], [t.records])
    compare(orc, th, t)


@pytest.mark.parametrize("i", [0, 1, 4, 6, 7, 8, 9])
def test_run_compression(i):
    """Run-compressed rows (Fig. 4) through
    thermo_query_runs against the oracle's runs."""
    t = SMALL[i]()
    orc, th = run_both(t)
    for k, obj in enumerate(t.objects):
        a, b = th.runs(obj[3]), orc.runs(k)
        for x, y in zip(a, b):
            assert np.array_equal(x, y), (t.name, obj[4])


def test_gemm_full_size_warp_records_from_host():
    """BJ configs[1] as 8.45 M warp-instruction records ingested from pinned host
    memory (several staged chunks): the closed forms on every cell."""
    from paper_2507_18729_b200 import Thermo
    t = tg.gemm(1024, 1024, 128, "v00", device="cuda")
    w = tg.to_warp_records(t.records)
    objects = t.objects
    del t
    host = torch.empty_like(w, device="cpu").pin_memory()
    host.copy_(w)
    del w
    th = Thermo(max_launches=1, max_warps_per_launch=1 << 20)
    th.register_objects(objects)
    th.ingest_warp(host)
    th.build()
    assert (th.heatmap(0, WORD) == 1024).all() and (th.heatmap(0, SECTOR) == 1024).all()
    assert (th.heatmap(1, WORD) == 32).all() and (th.heatmap(1, SECTOR) == 256).all()
    assert (th.heatmap(2, WORD) == 1).all() and (th.heatmap(2, SECTOR) == 8).all()
    st = th.stats()
    assert st["records"] == 270532608 and st["distinct_pairs"] == 22020096


def test_window_boundaries():
    """Objects and instructions across 4 GiB address windows (the fast decoder
    works on 32-bit offsets inside one window) and at the top of the 48-bit
    space; lanes of one instruction in two windows go to the general path."""
    import torch
    g = torch.Generator().manual_seed(17)
    objects = [(0xFFFFF000, 0x3000, 0, 1, "cross4G"), (0x2FFFFFFE0, 100, 0, 2, "cross8G"),
               (0x3FFFFFF00, 0x200, 0, 3, "cross16G"), ((1 << 48) - 4096, 4096 - 8, 0, 4, "top"),
               (0xFFFFF000, 0x2000, 1, 5, "shared-cross")]
    n_instr = 3000
    oi = torch.randint(0, len(objects), (n_instr,), generator=g)
    base = torch.tensor([o[0] for o in objects])[oi]
    ln = torch.tensor([o[1] for o in objects])[oi]
    space = torch.tensor([o[2] for o in objects])[oi]
    lane = torch.arange(32)
    mode = torch.randint(0, 3, (n_instr,), generator=g)
    start = (torch.rand(n_instr, generator=g) * (ln + 64).to(torch.float64)).to(torch.int64) - 32
    stride = torch.randint(1, 200, (n_instr,), generator=g)
    off = torch.where((mode == 0)[:, None], start[:, None] + 4 * lane[None, :],
                      torch.where((mode == 1)[:, None], start[:, None] + stride[:, None] * lane[None, :],
                                  (torch.rand((n_instr, 32), generator=g) * (ln + 64).to(torch.float64)[:, None]).to(
                                      torch.int64) - 32))
    addr = torch.clamp(base[:, None] + off, min=0, max=(1 << 48) - 16)
    active = torch.rand((n_instr, 32), generator=g) < 0.8
    active[:, 0] = True
    l2s = torch.randint(0, 4, (n_instr,), generator=g)
    warp = torch.randint(0, 40, (n_instr,), generator=g)
    recs = tg.from_instructions(addr, active, warp, 0x100 + 16 * (oi % 3), 0, l2s, space)
    t = tg.Trace("windows", objects, recs, meta=dict(launches=1))
    for dedup in (0, 1, 2):
        orc, th = run_both(t, dedup=dedup)
        compare(orc, th, t)
    # the same instructions as warp-instruction records
    from paper_2507_18729_b200 import Thermo
    th = gpu_ctx(t)
    th.ingest_warp(tg.to_warp_records(recs).cuda())
    th.build(BOTH)
    compare(oracle.run([o[:4] for o in objects], [recs]), th, t)


@pytest.mark.parametrize("dedup", [0, 1, 2])
def test_many_objects(dedup):
    """1000 registered objects (near THERMO_MAX_OBJECTS): the shared-memory object
    table, the binary searches and the interval cache at full size."""
    t = tg.random_trace(n=40000, seed=31, n_objects=1000, n_warps=200, n_launches=2, max_len=400)
    t.meta["launches"] = 2
    orc, th = run_both(t, dedup=dedup)
    compare(orc, th, t)
    from paper_2507_18729_b200 import Thermo
    objects, recs = tg.random_warp_trace(n_instr=3000, seed=32, n_objects=1000, max_len=400)
    tw = tg.Trace("warp-many", objects, recs, meta=dict(launches=2))
    th = Thermo(max_launches=2, max_warps_per_launch=1 << 22, dedup=dedup)
    th.register_objects(objects)
    th.ingest_warp(recs.cuda())
    th.build(BOTH)
    orc = oracle.Oracle([o[:4] for o in objects])
    orc.ingest_warp(recs)
    orc.build()
    compare(orc, th, tw)


@pytest.mark.parametrize("dedup", [1, 2, 3])
def test_synthetic_medium_all_outputs(dedup):
    """BJ configs[4]'s generator (64 objects, 8 launches, the 8 motifs) at a size
    the oracle finishes in seconds: every heat-map row, histogram, per-pc row,
    indicator and stat, bit-exact, in every dedup mode."""
    from paper_2507_18729_b200 import Thermo
    t = tg.synthetic(n_objects=64, n_launches=8, warps_per_launch=256, records_per_warp=256, size_shift=14)
    orc = oracle.run([o[:4] for o in t.objects], t.calls())
    th = Thermo(max_launches=8, max_warps_per_launch=256, max_pcs=64, dedup=dedup)
    th.register_objects(t.objects)
    th.ingest(t.records.cuda())
    th.build(BOTH)
    compare(orc, th, t)
    th.build(BOTH, 5)  # one launch (the paper's per-kernel map, G2)
    o5 = oracle.run([o[:4] for o in t.objects], t.calls(), 5)
    compare(o5, th, t)


def _distinct_sector_warp(t):
    """Distinct (global sector, warp) pairs of a single-launch trace of 4-byte
    aligned accesses, by brute force (torch.unique on the device; no library
    code): the sum of all sector counts."""
    r = t.records
    addr = (r[:, 0].to(torch.int64) & 0xFFFFFFFF) | ((r[:, 1].to(torch.int64) & 0xFFFF) << 32)
    bases = torch.tensor(sorted(o[0] for o in t.objects), device=r.device)
    oi = torch.searchsorted(bases, addr, right=True) - 1
    sec = (addr >> 5) - (bases[oi] >> 5) + oi * (1 << 36)  # object-qualified sector
    return int(torch.unique(sec * (1 << 22) + r[:, 2].to(torch.int64)).shape[0])


def _part_hash(x):
    """Sector-hash partition id in [0, 64) of absolute sector indices (numpy
    uint64/int64 or torch int64; the product stays below 2^63)."""
    return ((x & 0x7FFFFFFF) * 2654435761 >> 26) & 63


def _partition_exact(t, th, part=0):
    """SURVEY.md:691-692: the oracle, exact, on the 1/64 sector-hash partition
    `part` -- every (object, sector) whose absolute sector index hashes to it,
    touched or not -- fed the records touching those sectors (a sector's row
    depends only on them); every row of the partition compared with the GPU's.
    Returns (rows compared, largest sector count in the partition)."""
    oi_l, se_l, abs_l = [], [], []
    for k, ob in enumerate(t.objects):
        ns = (ob[1] + 31) // 32
        a = np.arange(ns, dtype=np.int64) + ob[0] // 32
        m = _part_hash(a) == part
        oi_l.append(np.full(int(m.sum()), k, dtype=np.uint32))
        se_l.append(np.nonzero(m)[0].astype(np.uint64))
    oi, se = np.concatenate(oi_l), np.concatenate(se_l)
    keep = []
    r = t.records
    for a in range(0, r.shape[0], 1 << 26):
        c = r[a:a + (1 << 26)]
        addr = (c[:, 0].to(torch.int64) & 0xFFFFFFFF) | ((c[:, 1].to(torch.int64) & 0xFFFF) << 32)
        size = torch.ones_like(addr) << ((c[:, 1].to(torch.int64) >> 16) & 7)
        m = (_part_hash(addr >> 5) == part) | (_part_hash((addr + size - 1) >> 5) == part)
        keep.append(c[m].cpu())
    sub = torch.cat(keep)
    orc = oracle.Oracle([o[:4] for o in t.objects])
    orc.restrict(oi, se)
    orc.ingest(sub)
    orc.build()
    ref = orc.sample(oi, se)
    for k, ob in enumerate(t.objects):
        rows = np.nonzero(oi == k)[0]
        if not len(rows):
            continue
        both = th.heatmap(ob[3], BOTH).reshape(-1, 9)
        got = both[se[rows].astype(np.int64)]
        bad = np.nonzero((got != ref[rows]).any(1))[0]
        assert len(bad) == 0, (ob[4], int(se[rows][bad[0]]), got[bad[0]], ref[rows][bad[0]])
    print(f"partition {part}: {len(oi)} sectors, {sub.shape[0]} records, max sector count {int(ref[:, 8].max())}")
    return len(oi), int(ref[:, 8].max())


def test_synthetic_full_size_partition():
    """BJ configs[4] at bench size on one GPU (one rank's slice of the 8-GPU job:
    2^15 warps x 8 launches x 2048 records = 2^29 records over 64 objects of
    4-512 MB): every row of the 1/64 sector-hash partition exactly against the
    oracle, plus the histogram invariants (level sums = n_words / n_sectors) on
    every object."""
    t = tg.synthetic(warps_per_launch=1 << 15, warp_range=(0, 1 << 15), device="cuda")
    assert t.n == 1 << 29
    from paper_2507_18729_b200 import Thermo
    th = Thermo(max_launches=8, max_warps_per_launch=1 << 15, max_pcs=64)
    th.register_objects(t.objects)
    th.ingest(t.records)
    th.build(BOTH)
    st = th.stats()
    assert st["records"] == 1 << 29 and st["invalid"] == 0
    for ob in t.objects:
        assert th.histogram(ob[3], WORD).sum() == (ob[1] + 3) // 4
        assert th.histogram(ob[3], SECTOR).sum() == (ob[1] + 31) // 32
    n, mx = _partition_exact(t, th, part=0)
    assert n > 100_000 and mx > 1


def test_spmv_full_size_partition():
    """BJ configs[3] at bench size (CSR SpMV on an R-MAT scale-24 matrix, 840.6 M
    records, the bench's launch configuration: AUTO = SEGMENT with its big-sector
    kernels): every row of the 1/64 sector-hash partition (1.1 M sectors of all
    five objects, hot x sectors included) exactly against the oracle, plus the
    histogram invariants on every object."""
    t = tg.spmv(24, 16, device="cuda")
    from paper_2507_18729_b200 import Thermo
    th = Thermo(max_launches=max(1, int(t.meta.get("launches", 1))),  # bench.py's configuration
                max_warps_per_launch=max(1, int(t.meta.get("warps", 1 << 20))), max_pcs=int(t.meta.get("pcs", 256)))
    th.register_objects(t.objects)
    th.ingest(t.records)
    th.build(BOTH)
    st = th.stats()
    assert st["invalid"] == 0 and st["distinct_pairs"] == _distinct_sector_warp(t)
    for ob in t.objects:
        assert th.histogram(ob[3], WORD).sum() == (ob[1] + 3) // 4
        assert th.histogram(ob[3], SECTOR).sum() == (ob[1] + 31) // 32
    n, mx = _partition_exact(t, th, part=0)
    assert n > 1_000_000
    assert mx >= 2048  # a big sector (>= 2048 keys): the big-sector kernels at full size


@pytest.mark.parametrize("dedup", [3, 1])
def test_launch_whitelist(dedup):
    """Kernel sampling by whitelist on the 8-launch
    synthetic trace, per-lane and warp-instruction records, alone and combined
    with a sampled block (DENSE): every output against the oracle with the same
    whitelist (pinned against the pre-filtered trace); clearing it traces all."""
    from paper_2507_18729_b200 import Thermo
    t = tg.synthetic(n_objects=16, n_launches=8, warps_per_launch=256, records_per_warp=256, size_shift=14)
    for wl, bw, blk in (([1, 4, 7], 0, 0), ([2], 0, 0), ([0, 3, 5], 64, 1)):
        kw = dict(block_warps=bw, block_id=blk) if bw else dict(dedup=dedup)
        th = Thermo(max_launches=8, max_warps_per_launch=256, max_pcs=64, **kw)
        th.register_objects(t.objects)
        th.set_launch_whitelist(wl)
        th.ingest(t.records.cuda())
        th.build(BOTH)
        orc = oracle.Oracle([o[:4] for o in t.objects])
        if bw:
            orc.block_scope(bw, blk)
        orc.launch_whitelist(wl)
        for c in t.calls():
            orc.ingest(c)
        orc.build()
        compare(orc, th, t)
        # the same through warp-instruction records
        th.reset()
        th.ingest_warp(tg.to_warp_records(t.records).cuda())
        th.build(BOTH)
        compare(orc, th, t)
    th.set_launch_whitelist([])
    th.reset()
    th.ingest(t.records.cuda())
    th.build(BOTH)
    orc = oracle.Oracle([o[:4] for o in t.objects])
    orc.block_scope(64, 1)
    for c in t.calls():
        orc.ingest(c)
    orc.build()
    compare(orc, th, t)
    with pytest.raises(Exception):
        th.set_launch_whitelist([8])  # >= max_launches
