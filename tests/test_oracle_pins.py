"""Pins for the CPU oracle (CPU only; no GPU).

The oracle (oracle/thermo_oracle.cpp) is checked against things other than
itself: the paper's worked examples (tests/golden/paper_examples.json), closed
forms of the synthetic workloads (tests/golden/closed_forms.json), the paper's
own bitmask analyzer, brute force with numpy, and invariants
(BJ north_star).
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import tracegen as tg
from tests import oracle_refs as R

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PAPER = json.load(open(os.path.join(GOLD, "paper_examples.json")))
CLOSED = json.load(open(os.path.join(GOLD, "closed_forms.json")))


def objs(t):
    return [o[:4] for o in t.objects]


def run(t, calls=None, launch_filter=oracle.ALL_LAUNCHES):
    return oracle.run(objs(t), calls if calls is not None else t.calls(), launch_filter)


def hist_dict(h):
    return {str(i): int(v) for i, v in enumerate(h) if v}


def labels_of(o, idx):
    return oracle.label_names(o.classify()[idx]["labels"])


# ---------------------------------------------------------------- paper examples
def test_fig3_discrimination():
    """Fig. 3: equal access counts, different temperatures."""
    for v in "ab":
        g = PAPER[f"fig3{v}"]
        t = tg.fig3(v)
        o = run(t)
        wc, sc = o.word_counts(0), o.sector_counts(0)
        assert (wc[:8] == g["word_temp"]).all()
        assert sc[0] == g["sector_temp"]
        # access counts (the baseline metric the paper argues against): the
        # oracle's access counts against the figure's values
        acc = o.access_counts(0)[:8]
        assert (acc == g["access_per_word"]).all() and acc.sum() == g["access_per_sector"]
    assert labels_of(run(tg.fig3("b")), 0) == ["FalseSharing"]
    assert labels_of(run(tg.fig3("a")), 0) == []


@pytest.mark.parametrize("W", [2, 3, 8])
def test_fig6_misalignment(W):
    """Fig. 6: 128 B at offset 16 -> 5 sectors, boundary
    sectors shared by two warps; aligned variant -> 4 sectors."""
    g = PAPER["fig6"]
    o = run(tg.fig6(W, 16))
    wc, sc = o.word_counts(0), o.sector_counts(0)
    assert set(np.unique(wc[wc > 0])) == {1}
    for s in range(len(sc)):
        exp = g["boundary_sector_warps"] if (s % 4 == 0 and 1 <= s <= 4 * (W - 1)) else \
            (g["interior_sector_warps"] if 0 <= s <= 4 * W else 0)
        assert sc[s] == exp, s
    ind = o.classify()[0]
    assert ind["instrs"] == W and ind["misaligned_instrs"] == W
    touched = [s for s in range(len(sc)) if sc[s]]
    assert len([s for s in touched if s <= 4]) == g["sectors_loaded"]
    ind0 = run(tg.fig6(W, 0)).classify()[0]
    assert ind0["misaligned_instrs"] == 0
    assert "Misaligned" in oracle.label_names(ind["labels"])


def test_table1_gemm():
    """Table I: gemm_v00 A Hot, B/C False shared; gemm_v01 B Hot."""
    t1 = PAPER["table1"]
    t = tg.gemm(64, 64, 16, "v00")
    o = run(t)
    for i, (_, _, _, _, name) in enumerate(t.objects):
        assert labels_of(o, i) == t1["gemm_v00"][name], name
    t = tg.gemm(64, 64, 16, "v01")
    o = run(t)
    assert labels_of(o, 1) == t1["gemm_v01"]["B"]
    assert all("FalseSharing" not in labels_of(o, i) for i in range(3))


def test_table1_other_kernels():
    t1 = PAPER["table1"]
    o = run(tg.strided_gather(64, 1024, 3))
    assert sorted(labels_of(o, 1)) == sorted(t1["gramschmidt_kernel3"]["q"])
    ind = o.classify()[1]
    assert ind["dom_gap"] == 1024 and ind["touched_words"] == 64   # one word per row
    o = run(tg.smem_thread_local())
    assert labels_of(o, 0) == t1["spt_TTMRankRBNnzKernelSM"]["Y_shr"]
    assert (o.word_counts(0) == PAPER["smem_abuse"]["word_temp"]).all()
    o = run(tg.smem_warp_broadcast())
    assert labels_of(o, 0) == t1["cuSZp"]["exel_sum"]


def test_table1_spmv_rowoffsets():
    """P:780 rowOffsets[r+1] loads 5 sectors instead of 4 -> Misaligned."""
    t = tg.spmv(scale=10, edgefactor=8)
    o = run(t)
    assert "Misaligned" in labels_of(o, 0)
    n = t.meta["n"]
    wc = o.word_counts(0)
    r = np.arange(n + 1)
    exp = np.where((r % 32 == 0) & (r > 0) & (r < n), 2, 1)
    assert (wc == exp).all()
    assert (o.word_counts(4) == 1).all()  # y
    # the ro[r+1] instructions: each full warp touches 5 sectors
    f = R.fields(t.records)
    heads = np.nonzero(f["istart"])[0]
    pcs = f["pc"][heads]
    ro1 = heads[pcs == 0x210]
    a = f["addr"][ro1[0]:ro1[0] + 32]
    assert len(set((a // 32).tolist())) == PAPER["spmv_rowoffsets"]["sectors_loaded"]


def test_hot_and_strided_examples():
    """P:404 hot = 32 warps; P:455 strided: one word per sector, temp 8."""
    dev = "cpu"
    lane = torch.arange(32)
    base = 0x90000
    # 32 warps each read all 8 words of 4 sectors -> hot
    A = torch.stack([base + 4 * (lane % 32) for _ in range(32)])
    rec = tg.from_instructions(A, torch.ones_like(A, dtype=torch.bool), torch.arange(32), 0x10, 0, 2)
    o = oracle.run([(base, 128, 0, 0)], [rec])
    assert (o.word_counts(0) == PAPER["hot"]["warps"]).all() and (o.sector_counts(0) == 32).all()
    assert labels_of(o, 0) == ["Hot"]
    # 8 warps read word 0 of every sector (stride 8 words = G15 reading of "7")
    A = torch.stack([base + 32 * lane for _ in range(8)])
    rec = tg.from_instructions(A, torch.ones_like(A, dtype=torch.bool), torch.arange(8), 0x10, 0, 2)
    o = oracle.run([(base, 32 * 32, 0, 0)], [rec])
    wc = o.word_counts(0).reshape(-1, 8)
    assert ((wc > 0).sum(1) == PAPER["strided"]["touched_words_per_sector"]).all()
    assert (wc[:, 0] == PAPER["strided"]["word_temp"]).all()
    ind = o.classify()[0]
    assert ind["dom_gap"] == 8 and "Strided" in oracle.label_names(ind["labels"])


def _cv(temps):
    """Population coefficient of variation of the nonzero word temperatures
    (numpy's std / mean, ddof = 0) -- computed from the DESIGNED temperatures,
    not from the oracle's output."""
    x = np.asarray(temps, dtype=np.float64)
    x = x[x > 0]
    return float(x.std() / x.mean())


@pytest.mark.parametrize("dist", ["bimodal", "uniform", "constant"])
def test_random_hot_s363(dist):
    """S:363 / P:404 Fig. 5(f): word temps varying 3..29 per sector, sectors hot.
    Nested warp sets give word j exactly temps[j] warps and a sector the max of
    its words (closed form).  The label is RandomHot iff the CV of the nonzero
    word temps exceeds random_hot_cv = 1/2, else Hot.  Bimodal
    3/29 draws (CV ~0.81) fire RandomHot; uniform 3..29 draws (CV ~0.487) stay
    below the default threshold and read Hot (G13); a constant 29 is
    the CV = 0 hot spot of P:404."""
    g = PAPER["random_hot"]
    T = tg.hot_temps(8192, dist, lo=g["word_temp_lo"], hi=g["word_temp_hi"]).numpy()
    t = tg.hot_spots(T)
    o = run(t)
    assert (o.word_counts(0) == T).all()
    assert (o.sector_counts(0) == T.reshape(-1, 8).max(1)).all()
    cv = _cv(T)
    ind = o.classify()[0]
    # indicator sums against the designed temperatures
    assert ind["touched_words"] == len(T) and ind["sum_x"] == int(T.sum())
    assert (ind["sum_x2_hi"] << 64 | ind["sum_x2_lo"]) == int((T.astype(object) ** 2).sum())
    smax = T.reshape(-1, 8).max(1)
    assert ind["hot_sectors"] == int((smax >= 16).sum())     # theta_hot = 16, sector = max word
    want = g["label"] if cv > g["random_hot_cv"] else "Hot"
    assert labels_of(o, 0) == [want]
    assert (dist == "bimodal") == (want == "RandomHot")


@pytest.mark.parametrize("lo,hi,want", [(16, 48, "Hot"), (16, 49, "RandomHot"), (16, 47, "Hot")])
def test_random_hot_cv_boundary(lo, hi, want):
    """Equal numbers of words at lo and hi warps: population CV = (hi-lo)/(hi+lo),
    exactly 1/2 at 16/48.  S:359 'exceeds' is strict, so CV = 1/2 reads Hot.
    The sample-std reading (ddof = 1) would give 0.500015 and flip the 16/48
    case; this pins the population reading of G13."""
    T = np.tile(np.array([lo, hi], dtype=np.int64), 4 * 2048)
    cv = _cv(T)
    assert (cv > 0.5) == (want == "RandomHot")
    o = run(tg.hot_spots(torch.from_numpy(T)))
    assert labels_of(o, 0) == [want]
    o2 = o.classify({"cv_num": 1, "cv_den": 3})   # a lower threshold flips 16/48 too
    assert oracle.label_names(o2[0]["labels"]) == ["RandomHot"]


@pytest.mark.parametrize("N", [64, 96, 128])
def test_stencil_closed_form_enumeration(N):
    """tests/closed_forms.py's reader enumeration of the column-mapped stencil
    (every word of `in` and `out`, every sector, both histograms, every per-PC
    row) equals the oracle exactly at small N; the GPU tests then use it on the
    full 8192^2 trace (BJ configs[2])."""
    from tests import closed_forms as C
    t = tg.stencil(N)
    o = run(t)
    w_in, s_in, w_out, s_out = C.stencil_counts(N)
    assert (o.word_counts(0) == w_in.numpy().reshape(-1)).all()
    assert (o.sector_counts(0) == s_in.numpy().reshape(-1)).all()
    assert (o.word_counts(1) == w_out.numpy().reshape(-1)).all()
    assert (o.sector_counts(1) == s_out.numpy().reshape(-1)).all()
    for k, (wc, sc) in enumerate(((w_in, s_in), (w_out, s_out))):
        assert (o.hist(k, False) == C.level_hist(wc).numpy()).all()
        assert (o.hist(k, True) == C.level_hist(sc).numpy()).all()
    rows = o.per_pc()
    assert [r[1] for r in rows] == list(C.STENCIL_PCS)
    for k, (_, _, hw, hs) in enumerate(rows):
        wm, sm = C.stencil_pc_cells(N, k)
        wc, sc = (w_in, s_in) if k < 5 else (w_out, s_out)
        assert (hw == C.level_hist(wc[wm]).numpy()).all() and (hs == C.level_hist(sc[sm]).numpy()).all()


# ---------------------------------------------------------------- closed forms
def test_tiny_b_closed_form():
    g = CLOSED["tiny_b"]
    o = run(tg.tiny("B"))
    j = np.arange(1024)
    s = np.arange(128)
    assert (o.word_counts(0) == np.where(j == 0, 8, np.where(j % 32 == 0, 2, 1))).all()
    assert (o.sector_counts(0) == np.where(s == 0, 8, np.where(s % 4 == 0, 2, 1))).all()
    assert hist_dict(o.hist(0, False)) == g["hist_word"]
    assert hist_dict(o.hist(0, True)) == g["hist_sector"]
    ind = o.classify()[0]
    assert ind["instrs"] == g["instrs"] and ind["misaligned_instrs"] == g["misaligned"]
    assert oracle.label_names(ind["labels"]) == g["labels"]
    rows = o.per_pc()
    assert [hex(r[1]) for r in rows] == ["0x10", "0x20", "0x30", "0x40"]
    for la, pc, hw, hs in rows:
        assert hist_dict(hw) == g["per_pc_word"][hex(pc)]
        assert hist_dict(hs) == g["per_pc_sector"][hex(pc)]


def test_tiny_a_streaming_is_one():
    """BJ invariant: a fully coalesced streaming trace yields count 1 everywhere."""
    o = run(tg.tiny("A"))
    assert (o.word_counts(0) == 1).all() and (o.sector_counts(0) == 1).all()


@pytest.mark.parametrize("M,N,K,variant", [(64, 64, 16, "v00"), (128, 64, 8, "v00"), (64, 128, 8, "v01")])
def test_gemm_closed_form(M, N, K, variant):
    t = tg.gemm(M, N, K, variant)
    o = run(t)
    if variant == "v00":
        assert (o.word_counts(0) == N).all() and (o.sector_counts(0) == N).all()
        assert (o.word_counts(1) == M // 32).all() and (o.sector_counts(1) == 8 * M // 32).all()
        assert (o.word_counts(2) == 1).all() and (o.sector_counts(2) == 8).all()
    else:  # v01: B row k, col c read by the warps whose lanes cover c: one per (by,ty)
        assert (o.word_counts(1) == M).all()
        assert (o.word_counts(2) == 1).all() and (o.sector_counts(2) == 1).all()
    assert o.stats()["records"] == 2 * M * N * K + 2 * M * N


def test_stencil_closed_form():
    N = 96
    o = run(tg.stencil(N))
    wc = o.word_counts(0).reshape(N, N)
    sc = o.sector_counts(0).reshape(N, N // 8)
    i = np.arange(N)[:, None]
    e = (i % 32 == 31).astype(int) + (i % 32 == 0).astype(int)
    # interior words (all five readers exist): rows 2..N-3, cols 2..N-3
    assert (wc[2:N - 2, 2:N - 2] == (3 + e)[2:N - 2]).all()
    # interior sectors: rows 2..N-3, sectors 1..N/8-2 (neighbour columns exist)
    assert (sc[2:N - 2, 1:N // 8 - 1] == (10 + 8 * e)[2:N - 2]).all()
    wo = o.word_counts(1).reshape(N, N)
    assert (wo[1:N - 1, 1:N - 1] == 1).all() and (wo[0] == 0).all()
    so = o.sector_counts(1).reshape(N, N // 8)
    assert (so[1:N - 1, 1:N // 8 - 1] == 8).all()
    assert "FalseSharing" in labels_of(o, 1)


# ---------------------------------------------------------------- independent algorithms
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_vs_paper_bitmask(seed):
    """One launch, warps < 64: oracle == the paper's own sector_history_map."""
    t = tg.random_trace(n=6000, seed=seed, n_warps=64, n_launches=1, invalid_frac=0.02)
    o = run(t)
    ref = R.paper_bitmask(t.records)
    checked = 0
    for k, (base, ln, sp, _i) in enumerate(objs(t)):
        wc, sc = o.word_counts(k), o.sector_counts(k)
        for s in range(len(sc)):
            m = ref.get((sp, base // 32 + s), [0] * 9)
            for b in range(8):
                if 8 * s + b < len(wc):
                    assert wc[8 * s + b] == m[b]
            # sector: the paper's 9th mask; identical here since no sector is split
            # between mapped and unmapped words (objects are 32-aligned, G9) unless
            # the object's length is not a multiple of 32 (tail words unmapped)
            if ln % 32 == 0 or s < len(sc) - 1:
                assert sc[s] == m[8]
            checked += 1
    assert checked > 100


@pytest.mark.parametrize("seed", [4, 5, 6, 7])
def test_oracle_vs_brute_force(seed):
    t = tg.random_trace(n=8000, seed=seed, n_warps=200, n_launches=3)
    calls = [(0, 3000), (3000, 8000)]
    calls_t = [t.records[a:b] for a, b in calls]
    for lf in (None, 1):
        o = run(t, calls_t, oracle.ALL_LAUNCHES if lf is None else lf)
        wc, sc = R.brute_counts(objs(t), t.records, lf)
        for k in range(len(t.objects)):
            assert (o.word_counts(k) == wc[k]).all()
            assert (o.sector_counts(k) == sc[k]).all()
        # misalignment counters by plain loops
        ref = R.brute_instructions(objs(t), t.records, calls)
        ind = o.classify()
        for k in range(len(t.objects)):
            exp = [0, 0]
            for (la, ob), v in ref.items():
                if ob == k and (lf is None or la == lf):
                    exp[0] += v[0]; exp[1] += v[1]
            assert [ind[k]["instrs"], ind[k]["misaligned_instrs"]] == exp


def test_stats_counts():
    t = tg.random_trace(n=5000, seed=9, invalid_frac=0.05)
    o = run(t)
    f = R.fields(t.records)
    st = o.stats()
    assert st["records"] == 5000 and st["invalid"] == int((~f["valid"]).sum())
    v = f["valid"]
    words = ((f["addr"][v] + f["size"][v] - 1) // 4 - f["addr"][v] // 4 + 1).sum()
    assert st["unmapped_words"] + st["mapped_word_accesses"] == words


# ---------------------------------------------------------------- invariants
def test_invariants_counts_bounds():
    t = tg.random_trace(n=10000, seed=11, n_warps=40, n_launches=2)
    o = run(t)
    f = R.fields(t.records)
    n_lw = len(np.unique((f["launch"][f["valid"]] << 32) | f["warp"][f["valid"]]))
    for k, (base, ln, sp, _i) in enumerate(objs(t)):
        wc, sc = o.word_counts(k).astype(np.int64), o.sector_counts(k).astype(np.int64)
        assert wc.max(initial=0) <= n_lw
        pad = np.zeros(8 * len(sc) - len(wc), np.int64)
        w8 = np.concatenate([wc, pad]).reshape(-1, 8)
        assert (sc >= w8.max(1)).all() and (sc <= np.minimum(w8.sum(1), n_lw)).all()
        assert o.hist(k, False).sum() == len(wc) and o.hist(k, True).sum() == len(sc)
        # level = bit_width (G10): histogram recomputed with int.bit_length
        h = np.bincount([int(x).bit_length() for x in wc], minlength=33)
        assert (h == o.hist(k, False)).all()


def test_invariant_permutation_chunking_duplication():
    t = tg.random_trace(n=6000, seed=12, instr_len=(1, 32))
    base = run(t)
    ref = [(base.word_counts(k), base.sector_counts(k)) for k in range(len(t.objects))]
    ind0 = base.classify()
    perm = tg.shuffle_instructions(t.records, seed=3)
    dup = torch.cat([t.records, t.records])
    split = [t.records[a:b] for a, b in tg.split_calls(t.n, t.records, 5)]
    for variant, calls in (("perm", [perm]), ("dup", [dup]), ("split", split)):
        o = run(t, calls)
        for k in range(len(t.objects)):
            assert (o.word_counts(k) == ref[k][0]).all(), variant
            assert (o.sector_counts(k) == ref[k][1]).all(), variant
        ind = o.classify()
        for k in range(len(t.objects)):
            for f in ("touched_sectors", "touched_words", "hot_sectors", "fs_sectors", "labels", "dom_gap"):
                assert ind[k][f] == ind0[k][f], (variant, f)


def test_invariant_monotone():
    t = tg.random_trace(n=4000, seed=13)
    a = run(t, [t.records[:2500]])
    b = run(t)
    for k in range(len(t.objects)):
        assert (a.word_counts(k) <= b.word_counts(k)).all()
        assert (a.sector_counts(k) <= b.sector_counts(k)).all()


def test_launch_filter_equals_prefiltered_trace():
    t = tg.random_trace(n=6000, seed=14, n_launches=4, instr_len=(1, 32))
    f = R.fields(t.records)
    for L in range(4):
        a = run(t, launch_filter=L)
        # instructions are single-launch in random_trace, so a prefiltered trace
        # has the same instruction structure
        b = run(t, [t.records[torch.from_numpy(f["launch"] == L)]])
        for k in range(len(t.objects)):
            assert (a.word_counts(k) == b.word_counts(k)).all()
            assert (a.sector_counts(k) == b.sector_counts(k)).all()
        assert [r[:2] for r in a.per_pc()] == [r[:2] for r in b.per_pc()]


def test_per_pc_brute_force():
    t = tg.random_trace(n=3000, seed=15, n_pcs=5)
    o = run(t)
    f = R.fields(t.records)
    wcs = [o.word_counts(k) for k in range(len(t.objects))]
    scs = [o.sector_counts(k) for k in range(len(t.objects))]
    sets = {}
    for i in np.nonzero(f["valid"])[0]:
        a, sz, sp = int(f["addr"][i]), int(f["size"][i]), int(f["space"][i])
        key = (int(f["launch"][i]), int(f["pc"][i]))
        for w in range(a // 4, (a + sz - 1) // 4 + 1):
            for k, (base, ln, osp, _i) in enumerate(objs(t)):
                if osp == sp and base <= 4 * w < base + ln:
                    sets.setdefault(key, set()).add((k, w - base // 4))
    rows = o.per_pc()
    assert [r[:2] for r in rows] == sorted(sets)
    for la, pc, hw, hs in rows:
        ws = sets[(la, pc)]
        ew = np.bincount([int(wcs[k][w]).bit_length() for k, w in ws], minlength=33)
        es = np.bincount([int(scs[k][s]).bit_length() for k, s in {(k, w // 8) for k, w in ws}], minlength=33)
        assert (hw == ew).all() and (hs == es).all()


def test_indicators_from_brute_counts():
    """T, TW, hot/fs sectors, sums and gap mode recomputed with numpy from the
    brute-force counts (not from the oracle's own arrays)."""
    t = tg.random_trace(n=12000, seed=16, n_warps=300, n_objects=4)
    o = run(t)
    wc_all, sc_all = R.brute_counts(objs(t), t.records)
    P = oracle.DEFAULT_PARAMS
    for k, ind in enumerate(o.classify()):
        wc, sc = wc_all[k].astype(np.int64), sc_all[k].astype(np.int64)
        pad = np.concatenate([wc, np.zeros(8 * len(sc) - len(wc), np.int64)]).reshape(-1, 8)
        mw = pad.max(1)
        t_ = sc > 0
        assert ind["touched_sectors"] == t_.sum() and ind["touched_words"] == (wc > 0).sum()
        hot = t_ & (sc >= P["theta_hot"]) & (4 * sc <= 5 * mw)
        fs = t_ & (sc >= 4 * mw) & (sc >= 4)
        assert ind["hot_sectors"] == hot.sum() and ind["fs_sectors"] == fs.sum()
        nz = wc[wc > 0]
        assert ind["sum_x"] == nz.sum()
        assert ind["sum_x2_lo"] + (ind["sum_x2_hi"] << 64) == int((nz.astype(object) ** 2).sum())
        pos = np.nonzero(wc)[0]
        gaps = np.diff(pos)
        assert ind["gaps"] == len(gaps)
        if len(gaps):
            vals, cnt = np.unique(gaps, return_counts=True)
            j = cnt.argmax()
            if 2 * cnt[j] > len(gaps):
                assert (ind["dom_gap"], ind["dom_count"]) == (vals[j], cnt[j])
            else:
                assert (ind["dom_gap"], ind["dom_count"]) == (0, 0)


@pytest.mark.parametrize("seed", [1, 2])
def test_access_counts_brute_force_and_bounds(seed):
    """Access counts: brute force over the records'
    touched words (all launches), and temperature <= accesses, equal zeros."""
    t = tg.random_trace(n=6000, seed=seed, n_launches=3)
    o = run(t, launch_filter=1)  # the launch filter does not apply to accesses
    f = R.fields(t.records)
    for k, (base, ln, space, _id, _l) in enumerate(t.objects):
        nw = (ln + 3) // 4
        ref = np.zeros(nw, dtype=np.int64)
        for a, sz, sp, ok in zip(f["addr"], f["size"], f["space"], f["valid"]):
            if not ok or sp != space:
                continue
            for w in range(a >> 2, ((a + sz - 1) >> 2) + 1):
                if base <= 4 * w < base + ln:
                    ref[w - base // 4] += 1
        acc = o.access_counts(k)
        assert np.array_equal(acc, ref)
        o_all = run(t)
        wc = o_all.word_counts(k)
        assert (wc <= acc).all() and ((wc == 0) == (acc == 0)).all()


@pytest.mark.parametrize("block", [0, 3])
def test_block_scope(block):
    """Sampled-block mode: the oracle's block
    scope equals the trace pre-filtered to that block's warps, and -- warp ids
    being < 64 inside one block -- the paper's own per-sector bitmask algorithm
     on those records."""
    t = tg.gemm(64, 64, 16, "v00")           # block 32x32: 32 warps per block
    o = oracle.Oracle(objs(t))
    o.block_scope(32, block)
    o.ingest(t.records)
    o.build()
    f = R.fields(t.records)
    keep = (f["warp"] // 32) == block
    sub = t.records[torch.from_numpy(np.nonzero(keep)[0])]
    assert sub.shape[0] > 0
    p = oracle.Oracle(objs(t))
    p.ingest(sub)
    p.build()
    loc = sub.clone()
    loc[:, 2] = loc[:, 2] % 32                # warp index inside the block
    ref = R.paper_bitmask(loc)
    for k, (base, ln, space, _id, _l) in enumerate(t.objects):
        assert np.array_equal(o.word_counts(k), p.word_counts(k))
        assert np.array_equal(o.sector_counts(k), p.sector_counts(k))
        sc = o.sector_counts(k)
        for s in range(len(sc)):
            want = ref.get((space, (base >> 5) + s), [0] * 9)
            assert sc[s] == want[8]


def _expand_warp_records(recs):
    """Independent Python expansion of warp-instruction records into per-lane
    records (thermo.h thermo_warp_record): active lanes in order, the first
    with instr_start; address bits >= 48 or reserved flags make a lane invalid."""
    a = np.ascontiguousarray(recs.numpy()).view(np.uint32).reshape(-1, 68)
    out = []
    for r in a:
        warp, site, active, flags = int(r[0]), int(r[1]), int(r[2]), int(r[3])
        first = True
        for l in range(32):
            if not (active >> l) & 1:
                continue
            addr = int(r[4 + 2 * l]) | (int(r[5 + 2 * l]) << 32)
            resv = 1 if (addr >> 48) or (flags >> 7) else 0
            af = (addr & ((1 << 48) - 1)) | ((flags & 7) << 48) | (((flags >> 3) & 3) << 51) | \
                 (((flags >> 5) & 3) << 53) | ((1 if first else 0) << 55) | (resv << 56)
            first = False
            out.append([af & 0xFFFFFFFF, af >> 32, warp, site])
    return torch.from_numpy(np.array(out, dtype=np.uint64).astype(np.uint32).view(np.int32).reshape(-1, 4))


def _same(o1, o2, nobj):
    for k in range(nobj):
        assert np.array_equal(o1.word_counts(k), o2.word_counts(k))
        assert np.array_equal(o1.sector_counts(k), o2.sector_counts(k))
    assert o1.classify() == o2.classify()
    assert o1.stats() == o2.stats()
    p1, p2 = o1.per_pc(), o2.per_pc()
    assert [(r[0], r[1]) for r in p1] == [(r[0], r[1]) for r in p2]
    for a, b in zip(p1, p2):
        assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_warp_records_equal_their_lane_expansion(seed):
    """Warp-instruction records: by definition the
    per-lane records of the active lanes; the oracle's ingest_warp against an
    independent expansion fed to the per-lane oracle."""
    objects, recs = tg.random_warp_trace(n_instr=1500, seed=seed, n_launches=2)
    ow = oracle.Oracle([o[:4] for o in objects])
    ow.ingest_warp(recs)
    ow.build()
    ol = oracle.Oracle([o[:4] for o in objects])
    ol.ingest(_expand_warp_records(recs))
    ol.build()
    _same(ow, ol, len(objects))


@pytest.mark.parametrize("make", [lambda: tg.tiny("B"), lambda: tg.gemm(64, 64, 16, "v00"), lambda: tg.stencil(64)])
def test_to_warp_records_roundtrip(make):
    """Uniform per-lane traces convert to warp records with the same heat map."""
    t = make()
    ow = oracle.Oracle(objs(t))
    ow.ingest_warp(tg.to_warp_records(t.records))
    ow.build()
    _same(ow, run(t), len(t.objects))


def test_runs_closed_forms_and_round_trip():
    """Run compression (Fig. 4): gemm_v00's A is
    one run of identical hot sectors, Fig. 3(b) one row; expanding the runs of
    random traces gives back the dense rows exactly; runs are maximal."""
    t = tg.gemm(64, 64, 16, "v00")
    o = run(t)
    st, ct, tp = o.runs(0)                       # A: every sector 64 warps (N = 64)
    assert len(st) == 1 and ct[0] == o.n_sectors(0) and (tp[0] == 64).all()
    st, ct, tp = run(tg.fig3("b")).runs(0)     # the shared sector, then the untouched rest
    assert list(tp[0]) == [1] * 8 + [8] and ct[0] == 1 and (len(st) == 1 or not tp[1:].any())
    for seed in (1, 2):
        r = tg.random_trace(n=5000, seed=seed)
        o = run(r)
        for k in range(len(r.objects)):
            st, ct, tp = o.runs(k)
            rows = np.repeat(tp, ct.astype(np.int64), axis=0)
            wc = o.word_counts(k)
            dense = np.zeros((o.n_sectors(k), 9), dtype=np.uint32)
            dense[:, :8].flat[:len(wc)] = wc
            dense[:, 8] = o.sector_counts(k)
            assert np.array_equal(rows, dense)
            assert (st == np.concatenate([[0], np.cumsum(ct)[:-1]])).all()
            assert all((tp[i] != tp[i + 1]).any() for i in range(len(tp) - 1))  # maximal


@pytest.mark.parametrize("seed", [11, 12])
def test_restricted_sample_equals_brute_force(seed):
    """Sampled mode (the full-size parity tests): the oracle restricted to a
    set of sectors builds only their rows; each equals the brute-force count
    (a sector's row depends only on the records touching it), with and
    without a launch filter, and unsampled sectors read 0."""
    t = tg.random_trace(n=8000, seed=seed, n_warps=200, n_launches=3)
    rng = np.random.default_rng(seed)
    oi, se = [], []
    for k, ob in enumerate(t.objects):
        ns = (ob[1] + 31) // 32
        pick = rng.choice(ns, min(ns, 12), replace=False)
        oi += [k] * len(pick)
        se += list(pick)
    oi, se = np.array(oi), np.array(se, dtype=np.uint64)
    for lf in (None, 2):
        o = oracle.Oracle(objs(t))
        o.restrict(oi, se)
        o.ingest(t.records)
        o.build(oracle.ALL_LAUNCHES if lf is None else lf)
        rows = o.sample(oi, se)
        wc, sc = R.brute_counts(objs(t), t.records, lf)
        for row, k, s in zip(rows, oi, se):
            s = int(s)
            nw = len(wc[k])
            exp = [int(wc[k][8 * s + b]) if 8 * s + b < nw else 0 for b in range(8)] + [int(sc[k][s])]
            assert list(row) == exp, (k, s)
        other = o.sample(np.array([0]), np.array([int(s) for s in range(100) if (0, s) not in set(zip(oi, se))][:1],
                                                 dtype=np.uint64))
        assert (other == 0).all()


def test_launch_whitelist():
    """Kernel sampling by whitelist: the oracle with a
    launch whitelist equals the oracle on the trace pre-filtered to those
    launches' records, for every output; an empty whitelist traces all."""
    t = tg.random_trace(n=20000, seed=21, n_warps=300, n_launches=6)
    f = R.fields(t.records)
    for wl in ([1, 4], [0], [5, 2, 3]):
        o = oracle.Oracle(objs(t))
        o.launch_whitelist(wl)
        o.ingest(t.records)
        o.build()
        keep = np.isin(f["launch"], wl)
        sub = t.records[torch.from_numpy(np.nonzero(keep)[0])]
        assert 0 < sub.shape[0] < t.records.shape[0]
        p = oracle.Oracle(objs(t))
        p.ingest(sub)
        p.build()
        for k in range(len(t.objects)):
            assert np.array_equal(o.word_counts(k), p.word_counts(k))
            assert np.array_equal(o.sector_counts(k), p.sector_counts(k))
            assert np.array_equal(o.hist(k, False), p.hist(k, False))
        assert o.classify() == p.classify()
        assert [(r[0], r[1]) for r in o.per_pc()] == [(r[0], r[1]) for r in p.per_pc()]
    a = oracle.Oracle(objs(t))
    a.launch_whitelist([])
    a.ingest(t.records)
    a.build()
    b = oracle.run(objs(t), [t.records])
    for k in range(len(t.objects)):
        assert np.array_equal(a.word_counts(k), b.word_counts(k))
