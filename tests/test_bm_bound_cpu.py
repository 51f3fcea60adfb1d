"""The indicator kernels' shortcut for the dominant gap (DESIGN.md §5 a7,
indicators.cu stitch): per tile a Boyer-Moore summary (c, n) of its gaps is
merged into the object's candidate, and the verify scan is skipped when
2 * U <= N, U = sum over tiles of (N_t + n_t) / 2 if c_t == candidate else
(N_t - n_t) / 2, plus the cross-tile gaps equal to the candidate.

These CPU checks pin the argument the skip rests on, on random gap sequences
(no GPU, no library code): a summary formed by cancelling pairs of different
values bounds every value's count that way, so (1) a strict majority is always
the merged candidate and (2) it is never skipped; and the in-sector table
(gaps between consecutive set bits of an 8-bit mask, voted in order) is such a
summary.
"""
import random

import pytest


def vote_merge(a, b):  # indicators.cu vote_merge: cancel pairs of different values
    (ac, an), (bc, bn) = a, b
    if an == 0:
        return b
    if bn == 0:
        return a
    if ac == bc:
        return (ac, an + bn)
    return (ac, an - bn) if an >= bn else (bc, bn - an)


def summary(values):
    s = (0, 0)
    for v in values:
        s = vote_merge(s, (v, 1))
    return s


def tree_summary(values):
    """The same, merged as a tree (warp / block reductions)."""
    parts = [(v, 1) for v in values] or [(0, 0)]
    while len(parts) > 1:
        parts = [vote_merge(parts[i], parts[i + 1]) if i + 1 < len(parts) else parts[i] for i in range(0, len(parts), 2)]
    return parts[0]


def bound(tiles, cand):
    """U for candidate cand from the tile summaries (cross gaps as 1-element tiles)."""
    u = 0
    for vals in tiles:
        c, n = tree_summary(vals)
        g = len(vals)
        u += (g + n) // 2 if (n and c == cand) else (g - n) // 2
    return u


@pytest.mark.parametrize("seed", range(40))
def test_bound_never_hides_a_majority(seed):
    rng = random.Random(seed)
    n_tiles = rng.randint(1, 12)
    tiles = []
    maj = rng.randint(1, 9)
    p_maj = rng.choice([0.3, 0.49, 0.5, 0.51, 0.6, 0.9])
    for _ in range(n_tiles):
        k = rng.randint(0, 40)
        tiles.append([maj if rng.random() < p_maj else rng.randint(1, 9) for _ in range(k)])
    flat = [v for t in tiles for v in t]
    # the object's summary: tile summaries merged
    s = (0, 0)
    for t in tiles:
        s = vote_merge(s, tree_summary(t))
    counts = {v: flat.count(v) for v in set(flat)}
    for v, f in counts.items():
        # every value's count is bounded by the tile summaries' bound
        assert f <= bound(tiles, v)
        if 2 * f > len(flat):  # a strict majority: the candidate, and not skipped
            assert s[0] == v and s[1] > 0
            assert 2 * bound(tiles, v) > len(flat)


def in_sector_summary(m):
    """indicators.cu s_bm[m]: gaps between consecutive set bits of m, voted in order."""
    bits = [b for b in range(8) if (m >> b) & 1]
    return summary([b2 - b1 for b1, b2 in zip(bits, bits[1:])])


def test_in_sector_table_is_a_pairing_summary():
    for m in range(256):
        bits = [b for b in range(8) if (m >> b) & 1]
        gaps = [b2 - b1 for b1, b2 in zip(bits, bits[1:])]
        c, n = in_sector_summary(m)
        assert n <= len(gaps) and c < 8 and n < 16  # fits the table's 4 + 4 bits
        for v in set(gaps):
            f = gaps.count(v)
            assert f <= ((len(gaps) + n) // 2 if (n and c == v) else (len(gaps) - n) // 2)
        # the 1-gaps the first pass counts by a popcount
        assert gaps.count(1) == bin(m & (m >> 1)).count("1")
