"""Independent formulations used to PIN the oracle (tests only).

* ``paper_bitmask``: the paper's own analyzer (§IV-B2): a map from
  sector tag to nine 64-bit warp bitmasks, ``|= 1 << warp_id`` into the word's
  slot and slot 8, then popcount at flush.  Valid for one launch, warp < 64.
* ``brute_counts``: expand every valid record into (object, word, warp) tuples
  with numpy and count distinct tuples with ``np.unique`` -- a different
  formulation from the oracle's per-word ``std::set``.
* ``brute_instructions``: per-instruction sector sets by Python loops.
"""
from __future__ import annotations

import numpy as np


def fields(records) -> dict:
    a = np.ascontiguousarray(records.cpu().numpy() if hasattr(records, "cpu") else records).view(np.uint32)
    a = a.reshape(-1, 4).astype(np.uint64)
    af = a[:, 0] | (a[:, 1] << np.uint64(32))
    addr = af & np.uint64((1 << 48) - 1)
    l2s = (af >> np.uint64(48)) & np.uint64(7)
    kind = (af >> np.uint64(51)) & np.uint64(3)
    space = (af >> np.uint64(53)) & np.uint64(3)
    istart = (af >> np.uint64(55)) & np.uint64(1)
    resv = af >> np.uint64(56)
    size = np.left_shift(np.uint64(1), np.minimum(l2s, np.uint64(4)))
    valid = (l2s <= 4) & (kind <= 2) & (space <= 2) & (resv == 0) & (addr + size <= np.uint64(1 << 48))
    site = a[:, 3]
    return dict(addr=addr.astype(np.int64), size=size.astype(np.int64), space=space.astype(np.int64),
                istart=istart.astype(bool), valid=valid, warp=a[:, 2].astype(np.int64),
                pc=((site & np.uint64(0xFFFFF)) << np.uint64(4)).astype(np.int64),
                launch=(site >> np.uint64(20)).astype(np.int64))


def brute_counts(objects, records, launch_filter=None):
    """Returns (word_counts[o], sector_counts[o]) as numpy arrays."""
    f = fields(records)
    keep = f["valid"]
    if launch_filter is not None:
        keep &= f["launch"] == launch_filter
    addr, size, space = f["addr"][keep], f["size"][keep], f["space"][keep]
    lw = (f["launch"][keep] << 32) | f["warp"][keep]
    words, warps, spaces = [], [], []
    w0 = addr // 4
    w1 = (addr + size - 1) // 4
    for d in range(5):
        m = w0 + d <= w1
        words.append((w0 + d)[m]); warps.append(lw[m]); spaces.append(space[m])
    words, warps, spaces = np.concatenate(words), np.concatenate(warps), np.concatenate(spaces)
    wc, sc = [], []
    for (base, ln, sp, _id) in [o[:4] for o in objects]:
        nw, ns = (ln + 3) // 4, (ln + 31) // 32
        m = (spaces == sp) & (words * 4 >= base) & (words * 4 < base + ln)
        loc = words[m] - base // 4
        pairs = np.unique(np.stack([loc, warps[m]], 1), axis=0) if m.any() else np.zeros((0, 2), np.int64)
        c = np.bincount(pairs[:, 0], minlength=nw).astype(np.uint32) if len(pairs) else np.zeros(nw, np.uint32)
        spairs = np.unique(np.stack([pairs[:, 0] // 8, pairs[:, 1]], 1), axis=0) if len(pairs) else pairs
        s = np.bincount(spairs[:, 0], minlength=ns).astype(np.uint32) if len(spairs) else np.zeros(ns, np.uint32)
        wc.append(c); sc.append(s)
    return wc, sc


def paper_bitmask(records):
    """sector_history_map of P:321-328: {(space, tag): [9 x uint64]}."""
    f = fields(records)
    hist = {}
    for i in np.nonzero(f["valid"])[0]:
        a, sz, sp, w = int(f["addr"][i]), int(f["size"][i]), int(f["space"][i]), int(f["warp"][i])
        assert w < 64
        for b in range(a, a + sz):            # every byte's word (G4)
            tag, off = b // 32, (b % 32) // 4  # P:324, G3
            m = hist.setdefault((sp, tag), [0] * 9)
            m[off] |= 1 << w
            m[8] |= 1 << w
    return {k: [bin(x).count("1") for x in v] for k, v in hist.items()}


def brute_instructions(objects, records, calls=None):
    """{(launch, object_index): [instrs, misaligned]} by plain loops (G24)."""
    f = fields(records)
    n = len(f["addr"])
    bounds = calls or [(0, n)]
    out = {}
    for lo, hi in bounds:
        heads, last = [], None
        for i in range(lo, hi):   # explicit heads, plus a split every 32 records (G24)
            if i == lo or f["istart"][i] or i - last == 32:
                heads.append(i)
                last = i
        heads.append(hi)
        for h0, h1 in zip(heads[:-1], heads[1:]):
            idx = [i for i in range(h0, h1) if f["valid"][i]]
            if not idx:
                continue
            first = idx[0]
            sp = int(f["space"][first])
            wb = (int(f["addr"][first]) // 4) * 4
            obj = None
            for k, o in enumerate(objects):
                if o[2] == sp and o[0] <= wb < o[0] + o[1]:
                    obj = k
                    break
            if obj is None:
                continue
            secs, lo_b, hi_b = set(), None, None
            for i in idx:
                a = (int(f["space"][i]) << 48) | int(f["addr"][i])
                e = a + int(f["size"][i]) - 1
                secs.update(range(a // 32, e // 32 + 1))
                lo_b = a if lo_b is None else min(lo_b, a)
                hi_b = e if hi_b is None else max(hi_b, e)
            key = (int(f["launch"][first]), obj)
            c = out.setdefault(key, [0, 0])
            c[0] += 1
            c[1] += int(len(secs) > -(-(hi_b - lo_b + 1) // 32))
    return out
