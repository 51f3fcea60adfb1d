"""Closed forms of synthetic workloads at any size (test infrastructure).

These enumerate, from the kernel's own index expressions, which warps read each
word -- they share no code with the oracle or the CUDA path and are pinned
against the oracle at small sizes (tests/test_oracle_pins.py) before the GPU
tests use them at full size.

Stencil (tracegen.stencil, column-mapped 5-point, block (32, 8)): thread (i, j)
with i = bx*32 + tx (row), j = by*8 + ty (column) is live iff 1 <= i, j <= N-2
(interior I); it reads in[i][j], in[i-1][j], in[i+1][j], in[i][j-1], in[i][j+1]
(pcs 0x300..0x340) and writes out[i][j] (pc 0x350).  Its warp is identified by
(i // 32, j).  So word (r, c) of `in` is read by the warps
    (r//32, c) [c], ((r+1)//32, c) [n], ((r-1)//32, c) [s], (r//32, c+1) [w], (r//32, c-1) [e]
each present iff its reading thread is live.  A word's count is the number of
distinct present warps; a sector's the number over its 8 words (G6).
"""
from __future__ import annotations

import torch

STENCIL_PCS = (0x300, 0x310, 0x320, 0x330, 0x340, 0x350)


def _codes_in(N: int, rows: torch.Tensor, cols: torch.Tensor):
    """[R, C, 5] warp codes (rowblock * N + col) of the readers of in[rows][cols]
    in the order c, n, s, w, e; -1 where absent."""
    r = rows[:, None].expand(-1, cols.shape[0])
    c = cols[None, :].expand(rows.shape[0], -1)

    def live(i, j):
        return (i >= 1) & (i <= N - 2) & (j >= 1) & (j <= N - 2)

    cand = [(r, c), (r + 1, c), (r - 1, c), (r, c + 1), (r, c - 1)]  # reading thread (i, j)
    out = []
    for i, j in cand:
        out.append(torch.where(live(i, j), (i // 32) * N + j, torch.full_like(i, -1)))
    return torch.stack(out, -1)


def _distinct(codes: torch.Tensor) -> torch.Tensor:
    """Number of distinct non-negative entries along the last dim."""
    s, _ = torch.sort(codes, dim=-1)
    new = torch.ones_like(s, dtype=torch.bool)
    new[..., 1:] = s[..., 1:] != s[..., :-1]
    return ((s >= 0) & new).sum(-1)


def stencil_counts(N: int, device="cpu", row_block: int = 256):
    """(word counts [N, N], sector counts [N, N/8]) of `in` and `out`, int32."""
    dev = torch.device(device)
    cols = torch.arange(N, device=dev)
    w_in = torch.empty((N, N), dtype=torch.int32, device=dev)
    s_in = torch.empty((N, N // 8), dtype=torch.int32, device=dev)
    for r0 in range(0, N, row_block):
        rows = torch.arange(r0, min(N, r0 + row_block), device=dev)
        codes = _codes_in(N, rows, cols)                                      # [R, N, 5]
        w_in[r0:r0 + rows.shape[0]] = _distinct(codes).to(torch.int32)
        sec = codes.reshape(rows.shape[0], N // 8, 8 * 5)
        s_in[r0:r0 + rows.shape[0]] = _distinct(sec).to(torch.int32)
    live_r = (torch.arange(N, device=dev) >= 1) & (torch.arange(N, device=dev) <= N - 2)
    w_out = (live_r[:, None] & live_r[None, :]).to(torch.int32)             # one writer per word
    s_out = w_out.reshape(N, N // 8, 8).sum(-1).to(torch.int32)             # distinct columns = warps
    return w_in, s_in, w_out, s_out


def stencil_pc_cells(N: int, k: int, device="cpu"):
    """(word mask [N, N], sector mask [N, N/8]) of the cells pc STENCIL_PCS[k]
    touches: object 0 (`in`) for k < 5, object 1 (`out`) for k = 5."""
    dev = torch.device(device)
    di, dj = (0, -1, 1, 0, 0, 0)[k], (0, 0, 0, -1, 1, 0)[k]
    i = torch.arange(N, device=dev)
    live = (i >= 1) & (i <= N - 2)
    # word (r, c) is touched iff thread (r - di, c - dj) is live
    rl = torch.zeros(N, dtype=torch.bool, device=dev)
    cl = torch.zeros(N, dtype=torch.bool, device=dev)
    rl[max(0, di):N + min(0, di)] = live[max(0, -di):N - max(0, di)]
    cl[max(0, dj):N + min(0, dj)] = live[max(0, -dj):N - max(0, dj)]
    wm = rl[:, None] & cl[None, :]
    return wm, wm.reshape(N, N // 8, 8).any(-1)


def level_hist(counts: torch.Tensor) -> torch.Tensor:
    """33-bin histogram of bit_width(count) (G10), in integer arithmetic:
    bit_width(c) = number of powers of two 1, 2, 4, ... that are <= c."""
    c = counts.reshape(-1).to(torch.int64)
    pw = torch.tensor([1 << k for k in range(33)], dtype=torch.int64, device=c.device)
    lv = torch.bucketize(c, pw, right=True)
    return torch.bincount(lv, minlength=33)
