"""Workload generators (see tracegen/__init__.py for the record layout).

Every generator evaluates the address expressions of a kernel (or of a worked
example) lane by lane and returns a Trace.  Cited listings: gemm_v00/v01
(Listing 1; P:651 swap), gramschmidt kernel3 (Listing 4,
P:729-737), spmv_csr (Listing 5), PASTA-like SMEM accumulator
(Listing 2), cuSZp-like warp broadcast, Fig. 3
(P:238-256), Fig. 6.  Synthetic shapes/sizes follow SURVEY §8(d).
"""
from __future__ import annotations

import math

import torch

from . import (KIND_LD, KIND_ST, KIND_ATOM, SPACE_GLOBAL, SPACE_SHARED, Trace,
               from_instructions, pack_records, splitmix64, _lsr)

MB2 = 2 << 20


def _align(x, a=MB2):
    return (x + a - 1) // a * a


def _seed_off(seed: int) -> int:
    """Map a seed to a non-negative int64 counter offset."""
    return (seed * 0x9E3779B97F4A7C15) % (1 << 62)


def _lanes(dev):
    return torch.arange(32, dtype=torch.int64, device=dev)


def _concat(parts, dev):
    if not parts:
        return torch.empty((0, 4), dtype=torch.int32, device=dev)
    return parts[0] if len(parts) == 1 else torch.cat(parts)


# --------------------------------------------------------------------------
# tiny vector-add-like trace (BJ configs[0])
# --------------------------------------------------------------------------
def tiny(variant: str = "B", device="cpu") -> Trace:
    """One 4 KB object x at 0x10000, 8 warps (one 256-thread block).

    Thread t handles i = t + 256k, k = 0..3.  tiny-B per element:
    pc 0x10 LD x[i]; 0x20 LD x[(i+1)%1024]; 0x30 LD x[0]; 0x40 ST x[i] (4 B).
    tiny-A keeps pcs 0x10 and 0x40 only (pure streaming).
    """
    dev = torch.device(device)
    base = 0x10000
    pcs = [0x10, 0x20, 0x30, 0x40] if variant == "B" else [0x10, 0x40]
    lane = _lanes(dev)
    addrs, warps, pcl, kinds = [], [], [], []
    for w in range(8):
        for k in range(4):
            i = 32 * w + lane + 256 * k
            for pc in pcs:
                if pc == 0x10 or pc == 0x40:
                    e = i
                elif pc == 0x20:
                    e = (i + 1) % 1024
                else:
                    e = torch.zeros_like(i)
                addrs.append(base + 4 * e)
                warps.append(w)
                pcl.append(pc)
                kinds.append(KIND_ST if pc == 0x40 else KIND_LD)
    A = torch.stack(addrs)
    rec = from_instructions(A, torch.ones_like(A, dtype=torch.bool),
                            torch.tensor(warps, device=dev), torch.tensor(pcl, device=dev),
                            torch.tensor(kinds, device=dev), 2)
    return Trace(f"tiny-{variant}", [(base, 4096, SPACE_GLOBAL, 0, "x")], rec,
                 meta=dict(warps=8))


# --------------------------------------------------------------------------
# paper worked examples
# --------------------------------------------------------------------------
def fig3(variant: str, device="cpu") -> Trace:
    """Fig. 3: (a) one warp, 8 lanes read words 0-7 of sector 0;
    (b) warps 0-7 each read one distinct word of sector 0."""
    dev = torch.device(device)
    base = 0x20000
    if variant == "a":
        addr = base + 4 * torch.arange(8, device=dev)
        warp = torch.zeros(8, dtype=torch.int64, device=dev)
        start = torch.zeros(8, dtype=torch.int64, device=dev)
        start[0] = 1
    else:
        addr = base + 4 * torch.arange(8, device=dev)
        warp = torch.arange(8, device=dev)
        start = torch.ones(8, dtype=torch.int64, device=dev)
    rec = pack_records(addr, 2, KIND_LD, SPACE_GLOBAL, start, warp, 0x80, 0)
    return Trace(f"fig3{variant}", [(base, 256, SPACE_GLOBAL, 0, "buf")], rec)


def fig6(n_warps: int = 2, offset: int = 16, device="cpu") -> Trace:
    """Fig. 6 generalised: warp w reads 128 B (32 lanes x 4 B)
    starting at byte offset + 128 w."""
    dev = torch.device(device)
    base = 0x40000
    lane = _lanes(dev)
    A = torch.stack([base + offset + 128 * w + 4 * lane for w in range(n_warps)])
    rec = from_instructions(A, torch.ones_like(A, dtype=torch.bool),
                            torch.arange(n_warps, device=dev), 0x90, KIND_LD, 2)
    size = _align(offset + 128 * n_warps + 128, 32)
    return Trace(f"fig6-{n_warps}-{offset}", [(base, size, SPACE_GLOBAL, 0, "buf")], rec)


# --------------------------------------------------------------------------
# gemm_v00 / gemm_v01 (Listing 1; block 32x32)
# --------------------------------------------------------------------------
def gemm(M=1024, N=1024, K=128, variant="v00", device="cpu", chunk_records=1 << 26, warp_limit=None,
         warp_range=None) -> Trace:
    """Naive SGEMM trace, one C element per thread, fp32 row-major.

    v00: C_row = bx*32 + tx, C_col = by*32 + ty (Listing 1).  v01 swaps them
    (P:651).  Per thread: K x (LD A[row*K+k], LD B[k*N+col]), LD C, ST C.
    Global warp = (bx + gridDim.x*by)*32 + ty.  Records = 2MNK + 2MN.
    """
    assert M % 32 == 0 and N % 32 == 0
    dev = torch.device(device)
    baseA = 0x7F0000000000
    baseB = _align(baseA + 4 * M * K)
    baseC = _align(baseB + 4 * K * N)
    objects = [(baseA, 4 * M * K, SPACE_GLOBAL, 0, "A"), (baseB, 4 * K * N, SPACE_GLOBAL, 1, "B"),
               (baseC, 4 * M * N, SPACE_GLOBAL, 2, "C")]
    gdx = M // 32 if variant == "v00" else N // 32
    n_warps = (M // 32) * (N // 32) * 32
    if warp_limit is not None:  # prefix of the trace (first warp_limit warps)
        n_warps = min(n_warps, warp_limit)
    w_lo, w_hi = 0, n_warps
    if warp_range is not None:  # the warps [lo, hi) of the trace (one rank's slice)
        w_lo, w_hi = max(0, warp_range[0]), min(n_warps, warp_range[1])
        w_hi = max(w_lo, w_hi)
    ipw = 2 * K + 2                       # instructions per warp
    n_rec = (w_hi - w_lo) * ipw * 32
    out = torch.empty((n_rec, 4), dtype=torch.int32, device=dev)
    lane = _lanes(dev)
    t = torch.arange(ipw, dtype=torch.int64, device=dev)
    k_of_t = torch.clamp(t // 2, max=K - 1)
    warps_per_chunk = max(1, chunk_records // (ipw * 32))
    pos = 0
    for w0 in range(w_lo, w_hi, warps_per_chunk):
        gw = torch.arange(w0, min(w_hi, w0 + warps_per_chunk), dtype=torch.int64, device=dev)
        b, ty = gw // 32, gw % 32
        bx, by = b % gdx, b // gdx
        if variant == "v00":
            row = (bx * 32)[:, None] + lane[None, :]          # [W, 32]
            col = (by * 32 + ty)[:, None].expand(-1, 32)
        else:
            row = (by * 32 + ty)[:, None].expand(-1, 32)
            col = (bx * 32)[:, None] + lane[None, :]
        row, col = row[:, None, :], col[:, None, :]            # [W, 1, 32]
        k = k_of_t[None, :, None]
        isA = ((t % 2 == 0) & (t < 2 * K))[None, :, None]
        isB = ((t % 2 == 1) & (t < 2 * K))[None, :, None]
        aA = baseA + 4 * (row * K + k)
        aB = baseB + 4 * (k * N + col)
        aC = baseC + 4 * (row * N + col)
        addr = torch.where(isA, aA, torch.where(isB, aB, aC))  # [W, ipw, 32]
        pc = torch.where(t < 2 * K, 0x100 + 0x10 * (t % 2), 0x120 + 0x10 * (t - 2 * K))
        kind = torch.where(t == 2 * K + 1, KIND_ST, KIND_LD)
        W = gw.shape[0]
        rec = from_instructions(addr.reshape(W * ipw, 32), torch.ones((W * ipw, 32), dtype=torch.bool, device=dev),
                                gw[:, None].expand(W, ipw).reshape(-1), pc.repeat(W), kind.repeat(W), 2)
        out[pos:pos + rec.shape[0]] = rec
        pos += rec.shape[0]
    assert pos == n_rec
    return Trace(f"gemm_{variant}-{M}x{N}x{K}", objects, out,
                 meta=dict(M=M, N=N, K=K, variant=variant, warps=n_warps, warp_range=(w_lo, w_hi)))


# --------------------------------------------------------------------------
# 2-D 5-point stencil, column-mapped
# --------------------------------------------------------------------------
def stencil(N=8192, device="cpu", chunk_records=1 << 26) -> Trace:
    """in/out fp32 N x N row-major.  i = bx*32 + tx (row), j = by*8 + ty (col),
    block (32, 8), global warp = (bx + (N/32)*by)*8 + ty.  Interior threads
    (1 <= i, j <= N-2) issue LD c, n, s, w, e then ST out; 6 (N-2)^2 records."""
    assert N % 32 == 0
    dev = torch.device(device)
    base_in = 0x7D0000000000
    base_out = _align(base_in + 4 * N * N)
    objects = [(base_in, 4 * N * N, SPACE_GLOBAL, 0, "in"), (base_out, 4 * N * N, SPACE_GLOBAL, 1, "out")]
    gdx = N // 32
    n_warps = (N // 32) * (N // 8) * 8
    n_rec = 6 * (N - 2) * (N - 2)
    out = torch.empty((n_rec, 4), dtype=torch.int32, device=dev)
    lane = _lanes(dev)
    di = torch.tensor([0, -1, 1, 0, 0, 0], dtype=torch.int64, device=dev)
    dj = torch.tensor([0, 0, 0, -1, 1, 0], dtype=torch.int64, device=dev)
    isout = torch.tensor([0, 0, 0, 0, 0, 1], dtype=torch.int64, device=dev)
    pcs = torch.tensor([0x300, 0x310, 0x320, 0x330, 0x340, 0x350], dtype=torch.int64, device=dev)
    kinds = torch.tensor([0, 0, 0, 0, 0, 1], dtype=torch.int64, device=dev)
    warps_per_chunk = max(1, chunk_records // (6 * 32))
    pos = 0
    for w0 in range(0, n_warps, warps_per_chunk):
        gw = torch.arange(w0, min(n_warps, w0 + warps_per_chunk), dtype=torch.int64, device=dev)
        W = gw.shape[0]
        b, ty = gw // 8, gw % 8
        bx, by = b % gdx, b // gdx
        i = (bx * 32)[:, None] + lane[None, :]                  # [W, 32]
        j = (by * 8 + ty)[:, None].expand(-1, 32)
        act = (i >= 1) & (i <= N - 2) & (j >= 1) & (j <= N - 2)
        ii = i[:, None, :] + di[None, :, None]
        jj = j[:, None, :] + dj[None, :, None]
        base = torch.where(isout == 1, base_out, base_in)[None, :, None]
        addr = base + 4 * (ii * N + jj)                        # [W, 6, 32]
        rec = from_instructions(addr.reshape(W * 6, 32), act[:, None, :].expand(W, 6, 32).reshape(W * 6, 32),
                                gw[:, None].expand(W, 6).reshape(-1), pcs.repeat(W), kinds.repeat(W), 2)
        out[pos:pos + rec.shape[0]] = rec
        pos += rec.shape[0]
    assert pos == n_rec
    return Trace(f"stencil-{N}", objects, out, meta=dict(N=N, warps=n_warps))


# --------------------------------------------------------------------------
# CSR SpMV on an R-MAT matrix (Listing 5)
# --------------------------------------------------------------------------
def rmat_csr(scale: int, edgefactor: int, seed: int = 0x5EED0004, device="cpu",
             abcd=(0.57, 0.19, 0.19, 0.05)):
    """Graph500 R-MAT edges (no vertex permutation), duplicates removed, rows
    sorted.  Randomness: counter-based splitmix64 keyed by (seed, edge, level).
    Returns (rowOffsets int64 [n+1], colIndices int64 [nnz])."""
    dev = torch.device(device)
    n = 1 << scale
    m = edgefactor * n
    a, b, c, _ = abcd
    ta, tb, tc = (int(x * (1 << 53)) for x in (a, a + b, a + b + c))
    keys = []
    step = max(1, (1 << 24) // scale)
    for e0 in range(0, m, step):
        e = torch.arange(e0, min(m, e0 + step), dtype=torch.int64, device=dev)
        row = torch.zeros_like(e)
        col = torch.zeros_like(e)
        for lvl in range(scale):
            r = splitmix64(e * scale + lvl + _seed_off(seed))
            u = _lsr(r, 11)
            rb = (u >= tb).to(torch.int64)                       # quadrants c, d
            cb = (((u >= ta) & (u < tb)) | (u >= tc)).to(torch.int64)  # b, d
            row = row | (rb << (scale - 1 - lvl))
            col = col | (cb << (scale - 1 - lvl))
        keys.append(torch.unique(row * n + col))
    key = torch.unique(torch.cat(keys))
    rows, cols = key // n, key % n
    counts = torch.bincount(rows, minlength=n)
    ro = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    ro[1:] = torch.cumsum(counts, 0)
    return ro, cols


def spmv(scale=15, edgefactor=16, seed=0x5EED0004, device="cpu", rows_per_chunk=1 << 20, row_range=None,
         max_records=None) -> Trace:
    """One thread per row, block 256 (global warp = r // 32).  Per row: LD ro[r],
    LD ro[r+1]; per nnz i: LD col[i], LD val[i], LD x[col[i]] (lanes inactive
    past their row length); then ST y[r].  Records = 3 nnz + 3 n.
    row_range=(lo, hi): only the rows [lo, hi) (multiples of 32: whole warps;
    one rank's slice of the job); max_records: stop after the first chunk that
    reaches it (a prefix of whole warps, for bounded CPU samples)."""
    dev = torch.device(device)
    ro, ci = rmat_csr(scale, edgefactor, seed, device)
    n = ro.shape[0] - 1
    nnz = ci.shape[0]
    b_ro = 0x7E0000000000
    b_ci = _align(b_ro + 4 * (n + 1))
    b_va = _align(b_ci + 4 * nnz)
    b_x = _align(b_va + 4 * nnz)
    b_y = _align(b_x + 4 * n)
    objects = [(b_ro, 4 * (n + 1), SPACE_GLOBAL, 0, "rowOffsets"), (b_ci, 4 * nnz, SPACE_GLOBAL, 1, "colIndices"),
               (b_va, 4 * nnz, SPACE_GLOBAL, 2, "values"), (b_x, 4 * n, SPACE_GLOBAL, 3, "x"),
               (b_y, 4 * n, SPACE_GLOBAL, 4, "y")]
    parts = []
    lo, hi = (0, n) if row_range is None else (max(0, row_range[0]), min(n, row_range[1]))
    assert lo % 32 == 0 and (hi % 32 == 0 or hi == n), "row ranges hold whole warps"
    done = 0
    for r0 in range(lo, hi, rows_per_chunk):
        if max_records is not None and done >= max_records:
            break
        r1 = min(hi, r0 + rows_per_chunk)
        r = torch.arange(r0, r1, dtype=torch.int64, device=dev)
        ln = ro[r0 + 1:r1 + 1] - ro[r0:r1]
        w = r // 32
        lane = r % 32
        wmax = torch.zeros(int(w[-1] - w[0]) + 1, dtype=torch.int64, device=dev)
        wmax.scatter_reduce_(0, w - w[0], ln, reduce="amax")
        ylast = 2 + 3 * wmax[w - w[0]]                      # instr index of ST y per row
        # per-row fixed records: ro[r], ro[r+1], y[r]
        f_addr = torch.stack([b_ro + 4 * r, b_ro + 4 * (r + 1), b_y + 4 * r], 1)
        f_ins = torch.stack([torch.zeros_like(r), torch.ones_like(r), ylast], 1)
        f_pc = torch.tensor([0x200, 0x210, 0x250], device=dev).expand(r.shape[0], 3)
        f_kind = torch.tensor([0, 0, 1], device=dev).expand(r.shape[0], 3)
        # nnz records: (row, i, j)
        rr = torch.repeat_interleave(r, ln)
        start = torch.repeat_interleave(ro[r0:r1], ln)
        idx = torch.arange(rr.shape[0], dtype=torch.int64, device=dev) - \
            torch.repeat_interleave(torch.cumsum(ln, 0) - ln, ln)
        e = start + idx
        colv = ci[e]
        n_addr = torch.stack([b_ci + 4 * e, b_va + 4 * e, b_x + 4 * colv], 1)
        n_ins = 2 + 3 * idx[:, None] + torch.arange(3, device=dev)[None, :]
        n_pc = torch.tensor([0x220, 0x230, 0x240], device=dev).expand(rr.shape[0], 3)
        n_kind = torch.zeros_like(n_pc)
        addr = torch.cat([f_addr.reshape(-1), n_addr.reshape(-1)])
        ins = torch.cat([f_ins.reshape(-1), n_ins.reshape(-1)])
        pc = torch.cat([f_pc.reshape(-1), n_pc.reshape(-1)])
        kind = torch.cat([f_kind.reshape(-1), n_kind.reshape(-1)])
        rowv = torch.cat([r[:, None].expand(-1, 3).reshape(-1), rr[:, None].expand(-1, 3).reshape(-1)])
        key = ((rowv // 32) << 32) | (ins << 5) | (rowv % 32)
        order = torch.argsort(key)
        addr, ins, pc, kind, rowv = addr[order], ins[order], pc[order], kind[order], rowv[order]
        wv = rowv // 32
        first = torch.ones_like(ins)
        first[1:] = ((ins[1:] != ins[:-1]) | (wv[1:] != wv[:-1])).to(torch.int64)
        parts.append(pack_records(addr, 2, kind, SPACE_GLOBAL, first, wv, pc, 0))
        done += parts[-1].shape[0]
    return Trace(f"spmv-s{scale}-ef{edgefactor}", objects, _concat(parts, dev),
                 meta=dict(n=n, nnz=nnz, scale=scale, edgefactor=edgefactor, rows=(lo, hi)))


# --------------------------------------------------------------------------
# test-only synthetic analogs (Table I rows)
# --------------------------------------------------------------------------
def strided_gather(NI=64, NJ=1024, k=3, device="cpu") -> Trace:
    """gramschmidt_kernel3 (Listing 4): j = bx*256 + tx; if (j > k && j < NJ):
    ST r[k*NJ+j]; for i: LD q[i*NJ+k], LD a[i*NJ+j]; for i: LD q[i*NJ+k],
    LD a[i*NJ+j], ST a[i*NJ+j].  q: one word per row, shared by all warps."""
    dev = torch.device(device)
    b_a = 0x7C0000000000
    b_q = _align(b_a + 4 * NI * NJ)
    b_r = _align(b_q + 4 * NI * NJ)
    objects = [(b_a, 4 * NI * NJ, SPACE_GLOBAL, 0, "a"), (b_q, 4 * NI * NJ, SPACE_GLOBAL, 1, "q"),
               (b_r, 4 * NJ * NJ, SPACE_GLOBAL, 2, "r")]
    lane = _lanes(dev)
    addrs, acts, warps, pcs, kinds = [], [], [], [], []
    for w in range(NJ // 32):
        j = 32 * w + lane
        act = (j > k) & (j < NJ)

        def emit(a, pc, kd):
            addrs.append(a); acts.append(act); warps.append(w); pcs.append(pc); kinds.append(kd)
        emit(b_r + 4 * (k * NJ + j), 0x400, KIND_ST)
        for i in range(NI):
            emit(torch.full_like(j, b_q + 4 * (i * NJ + k)), 0x410, KIND_LD)
            emit(b_a + 4 * (i * NJ + j), 0x420, KIND_LD)
        for i in range(NI):
            emit(torch.full_like(j, b_q + 4 * (i * NJ + k)), 0x430, KIND_LD)
            emit(b_a + 4 * (i * NJ + j), 0x440, KIND_LD)
            emit(b_a + 4 * (i * NJ + j), 0x450, KIND_ST)
    rec = from_instructions(torch.stack(addrs), torch.stack(acts), torch.tensor(warps, device=dev),
                            torch.tensor(pcs, device=dev), torch.tensor(kinds, device=dev), 2)
    return Trace(f"gramschmidt_k3-{NI}x{NJ}", objects, rec, meta=dict(NI=NI, NJ=NJ, k=k))


def smem_thread_local(blocks=4, iters=4, device="cpu") -> Trace:
    """PASTA-like (Listing 2): Y_shr[y_id], y_id = tidy*32 + tidx, block (32, 8).
    ST Y_shr[y_id]=0; iters x (LD, ST Y_shr[y_id]); LD Y_shr[y_id]; ST Y_val[x].
    Each block's SMEM window gets a distinct synthetic base (G21)."""
    dev = torch.device(device)
    b_sh = 0x1000
    win = 4 * 32 * 8
    b_y = 0x7B0000000000
    objects = [(b_sh, win * blocks, SPACE_SHARED, 0, "Y_shr"), (b_y, 4 * 256 * blocks, SPACE_GLOBAL, 1, "Y_val")]
    lane = _lanes(dev)
    addrs, warps, pcs, kinds, spaces = [], [], [], [], []
    for blk in range(blocks):
        for ty in range(8):
            gw = blk * 8 + ty
            sh = b_sh + blk * win + 4 * (ty * 32 + lane)

            def emit(a, pc, kd, sp):
                addrs.append(a); warps.append(gw); pcs.append(pc); kinds.append(kd); spaces.append(sp)
            emit(sh, 0x500, KIND_ST, SPACE_SHARED)
            for _ in range(iters):
                emit(sh, 0x510, KIND_LD, SPACE_SHARED)
                emit(sh, 0x520, KIND_ST, SPACE_SHARED)
            emit(sh, 0x530, KIND_LD, SPACE_SHARED)
            emit(b_y + 4 * (blk * 256 + ty * 32 + lane), 0x540, KIND_ST, SPACE_GLOBAL)
    A = torch.stack(addrs)
    rec = from_instructions(A, torch.ones_like(A, dtype=torch.bool), torch.tensor(warps, device=dev),
                            torch.tensor(pcs, device=dev), torch.tensor(kinds, device=dev), 2,
                            space=torch.tensor(spaces, device=dev))
    return Trace(f"smem_thread_local-{blocks}", objects, rec)


def smem_warp_broadcast(blocks=4, device="cpu") -> Trace:
    """cuSZp-like: lane 0 writes one SMEM word per warp
    (word = warp-in-block), all 32 lanes of that warp read it back."""
    dev = torch.device(device)
    b_sh = 0x8000
    win = 4 * 32
    objects = [(b_sh, win * blocks, SPACE_SHARED, 0, "exel_sum")]
    lane = _lanes(dev)
    addrs, acts, warps, pcs, kinds = [], [], [], [], []
    for blk in range(blocks):
        for wib in range(8):
            gw = blk * 8 + wib
            a = torch.full_like(lane, b_sh + blk * win + 4 * wib)
            addrs += [a, a]
            acts += [lane == 0, torch.ones_like(lane, dtype=torch.bool)]
            warps += [gw, gw]
            pcs += [0x600, 0x610]
            kinds += [KIND_ST, KIND_LD]
    rec = from_instructions(torch.stack(addrs), torch.stack(acts), torch.tensor(warps, device=dev),
                            torch.tensor(pcs, device=dev), torch.tensor(kinds, device=dev), 2,
                            space=SPACE_SHARED)
    return Trace(f"smem_warp_broadcast-{blocks}", objects, rec)


# --------------------------------------------------------------------------
# (random) hot spots: word temperatures drawn per word (Fig. 5(e)/(f);
# S:363 "word temps varying 3..29 per sector, sectors hot -> RandomHot")
# --------------------------------------------------------------------------
def hot_temps(n_sectors=8192, dist="bimodal", seed=0x5EED0006, lo=3, hi=29, device="cpu") -> torch.Tensor:
    """Designed word temperatures, int64 [8 n_sectors]: "bimodal" draws lo or hi
    per word (probability 1/2 each), "uniform" draws uniformly from lo..hi,
    "constant" is hi everywhere (the all-32-warps hot spot of P:404 when hi =
    32).  Counter-based (splitmix64 keyed by seed and word index)."""
    dev = torch.device(device)
    w = torch.arange(8 * n_sectors, dtype=torch.int64, device=dev)
    r = _lsr(splitmix64(w + _seed_off(seed)), 11)          # 53 random bits
    if dist == "bimodal":
        return torch.where((r & 1) == 1, hi, lo)
    if dist == "uniform":
        return lo + (r % (hi - lo + 1))
    if dist == "constant":
        return torch.full_like(w, hi)
    raise ValueError(dist)


def hot_spots(temps: torch.Tensor, base=0x7A0000000000, pc=0x700, device="cpu") -> Trace:
    """One global object of len(temps) words; word j is read by the warps
    0 .. temps[j]-1 (nested warp sets), so by construction word j's distinct-warp
    count is temps[j] and a sector's is the largest of its 8 words' temps.
    Warp w runs one 32-lane load per group of 32 consecutive words; lane l is
    active iff temps[32 g + l] > w (instructions with no active lane are not
    emitted).  Record order: warps ascending, groups ascending."""
    dev = torch.device(device)
    t = torch.as_tensor(temps, dtype=torch.int64, device=dev)
    nw = t.shape[0]
    G = (nw + 31) // 32
    tp = torch.zeros(G * 32, dtype=torch.int64, device=dev)
    tp[:nw] = t
    W = int(tp.max())
    wv = torch.arange(W, dtype=torch.int64, device=dev)[:, None, None]          # [W, 1, 1]
    j = torch.arange(G * 32, dtype=torch.int64, device=dev).reshape(1, G, 32)    # [1, G, 32]
    act = (tp.reshape(1, G, 32) > wv).reshape(W * G, 32)
    A = (base + 4 * j).expand(W, G, 32).reshape(W * G, 32)
    keep = act.any(1)
    warp = wv.expand(W, G, 1).reshape(W * G)
    rec = from_instructions(A[keep], act[keep], warp[keep], pc, KIND_LD, 2)
    return Trace(f"hot_spots-{nw}", [(base, 4 * nw, SPACE_GLOBAL, 0, "x")], rec, meta=dict(warps=W))


# --------------------------------------------------------------------------
# random fuzz traces (brute-force pins, fuzz parity)
# --------------------------------------------------------------------------
def random_trace(n=20000, seed=1, n_objects=5, n_warps=50, n_launches=3, n_pcs=7,
                 invalid_frac=0.01, unmapped_frac=0.05, shared_frac=0.2, device="cpu",
                 instr_len=(1, 40), max_len=3000) -> Trace:
    """Random unaligned/straddling records of sizes 1/2/4/8/16 over random
    objects (global and shared), some unmapped and some invalid records, random
    instruction lengths (including > 32 records)."""
    g = torch.Generator().manual_seed(seed)

    def ri(lo, hi, size):
        return torch.randint(lo, hi, size, generator=g, dtype=torch.int64)

    objects = []
    bases = {0: 0x100000, 1: 0x2000}
    for o in range(n_objects):
        space = 1 if (o % 5 == 4 or torch.rand(1, generator=g).item() < shared_frac) else 0
        ln = int(ri(1, max_len, (1,)))
        base = bases[space] + 32 * int(ri(0, 4, (1,)))
        objects.append((base, ln, space, 100 + o, f"o{o}"))
        bases[space] = _align(base + ln + 1, 32) + 32 * int(ri(0, 3, (1,)))
    oi = ri(0, n_objects, (n,))
    base = torch.tensor([o[0] for o in objects])[oi]
    ln = torch.tensor([o[1] for o in objects])[oi]
    space = torch.tensor([o[2] for o in objects])[oi]
    off = (torch.rand(n, generator=g) * (ln + 40).to(torch.float64)).to(torch.int64) - 20
    unm = torch.rand(n, generator=g) < unmapped_frac
    off = torch.where(unm, ln + 64 + ri(0, 1000, (n,)), off)
    addr = torch.clamp(base + off, min=0)
    log2size = ri(0, 5, (n,))
    kind = ri(0, 3, (n,))
    # instruction structure: runs of random length share warp/pc/launch
    lens = ri(instr_len[0], instr_len[1] + 1, (n,))
    starts = torch.cumsum(lens, 0) - lens
    starts = starts[starts < n]
    istart = torch.zeros(n, dtype=torch.int64)
    istart[starts] = 1
    iid = torch.cumsum(istart, 0) - 1
    warp = ri(0, n_warps, (len(starts),))[iid]
    launch = ri(0, n_launches, (len(starts),))[iid]
    pc = (ri(1, n_pcs + 1, (len(starts),)) * 16)[iid]
    rec = pack_records(addr, log2size, kind, space, istart, warp, pc, launch)
    bad = torch.nonzero(torch.rand(n, generator=g) < invalid_frac).flatten()
    if len(bad):
        # corrupt: reserved bits, size code 5..7 or kind 3 / space 3
        which = ri(0, 3, (len(bad),))
        hi = rec[bad, 1].to(torch.int64) & 0xFFFFFFFF
        hi = torch.where(which == 0, hi | (1 << 24), torch.where(which == 1, hi | (7 << 16), hi | (3 << 19)))
        rec[bad, 1] = torch.where(hi >= (1 << 31), hi - (1 << 32), hi).to(torch.int32)
    return Trace(f"random-{n}-{seed}", objects, rec.to(device),
                 meta=dict(warps=n_warps, launches=n_launches))


def random_warp_trace(n_instr=3000, seed=1, n_objects=5, n_warps=60, n_launches=2, n_pcs=5, device="cpu",
                      max_len=3000):
    """Random warp-instruction records (thermo_warp_record): random active
    masks (empty and full included), sizes 1-16 B at random offsets (unaligned,
    straddling), addresses inside, near and outside the objects, some invalid
    flags / address bits >= 48.  Returns (Trace-like objects, int32 [n, 68])."""
    from . import pack_warp_records
    g = torch.Generator().manual_seed(seed)

    def ri(lo, hi, size):
        return torch.randint(lo, hi, size, generator=g, dtype=torch.int64)

    objects = []
    bases = {0: 0x100000, 1: 0x2000}
    for o in range(n_objects):
        space = 1 if o % 4 == 3 else 0
        ln = int(ri(1, max_len, (1,)))
        base = bases[space] + 32 * int(ri(0, 4, (1,)))
        objects.append((base, ln, space, 200 + o, f"w{o}"))
        bases[space] = _align(base + ln + 1, 32) + 32 * int(ri(0, 3, (1,)))
    I = n_instr
    oi = ri(0, n_objects, (I,))
    base = torch.tensor([o[0] for o in objects])[oi]
    ln = torch.tensor([o[1] for o in objects])[oi]
    space = torch.tensor([o[2] for o in objects])[oi]
    l2s = ri(0, 5, (I,))
    kind = ri(0, 3, (I,))
    mode = ri(0, 4, (I,))   # 0 contiguous, 1 strided, 2 random, 3 broadcast
    lane = torch.arange(32, dtype=torch.int64)
    start = (torch.rand(I, generator=g) * (ln + 40).to(torch.float64)).to(torch.int64) - 20
    stride = ri(1, 300, (I,))
    rnd = (torch.rand((I, 32), generator=g) * (ln + 64).to(torch.float64)[:, None]).to(torch.int64) - 32
    off = torch.where((mode == 0)[:, None], start[:, None] + lane[None, :] * (1 << l2s)[:, None],
          torch.where((mode == 1)[:, None], start[:, None] + lane[None, :] * stride[:, None],
          torch.where((mode == 2)[:, None], rnd, start[:, None].expand(I, 32))))
    addr = torch.clamp(base[:, None] + off, min=0)
    hi_bad = torch.rand((I, 32), generator=g) < 0.002
    addr = torch.where(hi_bad, addr | (1 << 50), addr)
    am = torch.rand(I, generator=g)
    active = torch.rand((I, 32), generator=g) < am[:, None]
    active[ri(0, I, (I // 20,))] = True
    active[ri(0, I, (I // 40,))] = False
    warp = ri(0, n_warps, (I,))
    launch = ri(0, n_launches, (I,))
    pc = ri(1, n_pcs + 1, (I,)) * 16
    flags = l2s | (kind << 3) | (space << 5)
    bad = torch.rand(I, generator=g) < 0.01
    flags = torch.where(bad, flags | (1 << 7), flags)
    flags = torch.where(torch.rand(I, generator=g) < 0.01, (flags & ~7) | 6, flags)  # size code 6: invalid
    recs = pack_warp_records(addr, active, warp, (pc >> 4) | (launch << 20), flags)
    return objects, recs.to(device)


# --------------------------------------------------------------------------
# synthetic multi-kernel trace over 64 objects
# --------------------------------------------------------------------------
def synthetic(n_objects=64, n_launches=8, warps_per_launch=1 << 18, records_per_warp=2048,
              seed=0x5EED0005, device="cpu", size_shift=22, launch_lo=0, launch_hi=None,
              warp_range=None) -> Trace:
    """Each launch touches 8 objects with one motif each (coalesced 4 B, float4,
    broadcast-hot, column-strided, stencil-halo, Zipf-like gather, +16 B
    misaligned stream, random atomics); object sizes 2^(size_shift + h mod 8) B.
    Warps issue records_per_warp/32 instructions cycling over the 8 motifs.
    Randomness: splitmix64 keyed by (seed, launch, warp, instruction, lane).
    warp_range=(lo, hi): only warps [lo, hi) of every launch (a rank's slice
    of the job, or a bounded sample); records are written into one
    preallocated tensor, so the peak is the trace plus one 2^24-record chunk."""
    dev = torch.device(device)
    sizes, bases, objects = [], [], []
    base = 0x600000000000
    for o in range(n_objects):
        h = int(splitmix64(torch.tensor([seed * 131 + o])).item()) & 0xFFFF
        sz = 1 << (size_shift + h % 8)
        objects.append((base, sz, SPACE_GLOBAL, o, f"obj{o}"))
        sizes.append(sz)
        bases.append(base)
        base = _align(base + sz)
    sizes_t = torch.tensor(sizes, dtype=torch.int64, device=dev)
    bases_t = torch.tensor(bases, dtype=torch.int64, device=dev)
    ipw = records_per_warp // 32
    lane = _lanes(dev)
    launch_hi = n_launches if launch_hi is None else launch_hi
    wlo, whi = (0, warps_per_launch) if warp_range is None else warp_range
    out = torch.empty(((launch_hi - launch_lo) * (whi - wlo) * records_per_warp, 4), dtype=torch.int32, device=dev)
    pos = 0
    wchunk = max(1, (1 << 24) // records_per_warp)
    for L in range(launch_lo, launch_hi):
        objs_L = torch.tensor([(L * 8 + m * 9) % n_objects for m in range(8)], dtype=torch.int64, device=dev)
        for w0 in range(wlo, whi, wchunk):
            w = torch.arange(w0, min(whi, w0 + wchunk), dtype=torch.int64, device=dev)
            W = w.shape[0]
            t = torch.arange(ipw, dtype=torch.int64, device=dev)
            motif = (t % 8)[None, :, None].expand(W, ipw, 32)
            o = objs_L[motif]
            osz = sizes_t[o]
            ob = bases_t[o]
            nwords = osz // 4
            it = (t // 8)[None, :, None]
            gw = w[:, None, None]
            rnd = splitmix64(_seed_off(seed + L) + (gw << 20) + (t[None, :, None] << 5) + lane[None, None, :])
            r31 = _lsr(rnd, 33)
            tid = gw * 32 + lane[None, None, :]
            coal = (tid * 4 + it * warps_per_launch * 128) % osz
            f4 = (tid * 16 + it * warps_per_launch * 512) % osz
            hot = ((it * 4) % 4096) + torch.zeros_like(tid)
            colstr = ((lane[None, None, :] * 1024 + gw + it * 7) * 4) % osz
            halo = ((tid + (t[None, :, None] % 3 - 1) * 1024) * 4) % osz
            zipf = ((r31 % 1024) * (r31 % 1024) % 65536) * 4 % osz
            mis = (tid * 4 + 16 + it * warps_per_launch * 128) % (osz - 16)
            rnd_a = (r31 % nwords) * 4
            off = torch.stack([coal, f4, hot, colstr, halo, zipf, mis, rnd_a], 0)
            off = torch.gather(off, 0, motif[None]).squeeze(0)
            addr = ob + (off // 4) * 4
            l2s = torch.where(motif == 1, 4, 2)
            kind = torch.where(motif == 7, KIND_ATOM, torch.where(motif == 0, KIND_ST, KIND_LD))
            pc = 0x1000 + 0x10 * motif
            first = torch.zeros_like(addr)
            first[:, :, 0] = 1
            rec = pack_records(addr.reshape(-1), l2s.reshape(-1), kind.reshape(-1), SPACE_GLOBAL,
                               first.reshape(-1), gw.expand(W, ipw, 32).reshape(-1), pc.reshape(-1), L)
            out[pos:pos + rec.shape[0]] = rec
            pos += rec.shape[0]
            del rec, addr, off, rnd, r31
    return Trace(f"synthetic-{n_objects}x{n_launches}", objects, out,
                 meta=dict(launches=n_launches, warps=warps_per_launch, pcs=8 * n_launches))


WORKLOADS = {
    "tiny": lambda device="cpu": tiny("B", device),
    "sgemm": lambda device="cpu": gemm(1024, 1024, 128, "v00", device),
    "stencil": lambda device="cpu": stencil(8192, device),
    "spmv": lambda device="cpu": spmv(24, 16, device=device),
}
