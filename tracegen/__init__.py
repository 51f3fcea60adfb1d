"""Seeded, synthetic memory-access trace generators (test + bench infrastructure).

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NO arithmetic of the heat-map method (no sector tags, word masks,
distinct-warp counting, levels or pattern rules): it only evaluates the address
expressions of the application kernels the paper studies (Listings 1, 4, 5;
P:629-637) plus the worked examples of Figs. 3/5/6, and
packs each active lane's access into the 16-byte record of include/thermo.h:

    u64 addr_flags : [0,48) byte address | [48,51) log2(size) | [51,53) kind
                     | [53,55) space | [55] instr_start | [56,64) reserved = 0
    u32 warp       : global warp id within its launch
    u32 site       : [0,20) pc >> 4 | [20,32) launch id

Records are built with torch integer ops so the same generator runs on the CPU
(for the oracle) and on the GPU (for the bench), giving identical bytes.
Default record order: blocks in linear order, warps ascending, program
order within a warp, lanes ascending; `shuffle_instructions` gives the seeded
warp-instruction-granularity permutation variant.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

KIND_LD, KIND_ST, KIND_ATOM = 0, 1, 2
SPACE_GLOBAL, SPACE_SHARED, SPACE_LOCAL = 0, 1, 2
MASK64 = (1 << 64) - 1


@dataclass
class Trace:
    name: str
    objects: list            # [(base, len, space, id, label)]
    records: torch.Tensor    # int32 [n, 4] (16-byte records)
    chunks: list = field(default_factory=list)  # ingest-call boundaries [(lo, hi)]
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.records.shape[0])

    def calls(self):
        """Record slices, one per ingest call."""
        if not self.chunks:
            return [self.records]
        return [self.records[lo:hi] for lo, hi in self.chunks]


def _u32_to_i32(x: torch.Tensor) -> torch.Tensor:
    x = x.to(torch.int64)
    return torch.where(x >= (1 << 31), x - (1 << 32), x).to(torch.int32)


def pack_records(addr, log2size, kind, space, istart, warp, pc, launch) -> torch.Tensor:
    """Pack per-record fields (int64 tensors, broadcastable) into int32 [n, 4]."""
    addr = addr.to(torch.int64)
    n = addr.shape[0]
    dev = addr.device

    def b(v):
        v = torch.as_tensor(v, dtype=torch.int64, device=dev)
        return v.expand(n) if v.dim() == 0 else v.to(torch.int64)

    hi = (addr >> 32) | (b(log2size) << 16) | (b(kind) << 19) | (b(space) << 21) | (b(istart) << 23)
    lo = addr & 0xFFFFFFFF
    site = (b(pc) >> 4) | (b(launch) << 20)
    out = torch.empty((n, 4), dtype=torch.int32, device=dev)
    out[:, 0] = _u32_to_i32(lo)
    out[:, 1] = _u32_to_i32(hi)
    out[:, 2] = _u32_to_i32(b(warp))
    out[:, 3] = _u32_to_i32(site)
    return out


def from_instructions(lane_addr, active, warp, pc, kind, log2size, space=0, launch=0) -> torch.Tensor:
    """Warp-level instructions -> per-lane records (inactive lanes dropped).

    lane_addr, active: [I, 32];  warp, pc, kind, log2size, space, launch: [I] or
    scalars.  The first active lane of each instruction carries instr_start.
    """
    I = lane_addr.shape[0]
    dev = lane_addr.device

    def col(v):
        v = torch.as_tensor(v, dtype=torch.int64, device=dev)
        return (v.expand(I) if v.dim() == 0 else v).unsqueeze(1).expand(I, 32)

    active = active.to(torch.bool)
    first = active & (torch.cumsum(active.to(torch.int32), dim=1) == 1)
    sel = active.reshape(-1)
    return pack_records(
        lane_addr.reshape(-1)[sel], col(log2size).reshape(-1)[sel], col(kind).reshape(-1)[sel],
        col(space).reshape(-1)[sel], first.reshape(-1)[sel].to(torch.int64),
        col(warp).reshape(-1)[sel], col(pc).reshape(-1)[sel], col(launch).reshape(-1)[sel])


def pack_warp_records(lane_addr, active, warp, site, flags) -> torch.Tensor:
    """Warp-instruction records (include/thermo.h thermo_warp_record, 272 B =
    int32 [I, 68]): warp, site, active mask, flags, then 32 u64 lane addresses.
    lane_addr int64 [I, 32]; active bool [I, 32]; warp/site/flags int64 [I]."""
    I = lane_addr.shape[0]
    dev = lane_addr.device
    out = torch.zeros((I, 68), dtype=torch.int32, device=dev)
    bits = (active.to(torch.int64) << torch.arange(32, device=dev, dtype=torch.int64)).sum(1)
    out[:, 0] = _u32_to_i32(torch.as_tensor(warp, device=dev).to(torch.int64).expand(I))
    out[:, 1] = _u32_to_i32(torch.as_tensor(site, device=dev).to(torch.int64).expand(I))
    out[:, 2] = _u32_to_i32(bits)
    out[:, 3] = _u32_to_i32(torch.as_tensor(flags, device=dev).to(torch.int64).expand(I))
    a = lane_addr.to(torch.int64)
    out[:, 4::2] = _u32_to_i32(a & 0xFFFFFFFF)
    out[:, 5::2] = _u32_to_i32((a >> 32) & 0xFFFFFFFF)
    return out


def to_warp_records(records: torch.Tensor) -> torch.Tensor:
    """Per-lane records -> warp-instruction records, one per instruction (its
    records become lanes 0..len-1).  Every instruction must be <= 32 records
    with one warp, site, size, kind and space, and no reserved bits."""
    r = records.to(torch.int64) & 0xFFFFFFFF
    n = r.shape[0]
    dev = records.device
    hi = r[:, 1]
    head = ((hi >> 23) & 1).bool()
    head[0] = True
    iid = torch.cumsum(head.to(torch.int64), 0) - 1
    hidx = torch.nonzero(head).flatten()
    pos = torch.arange(n, device=dev) - hidx[iid]
    assert int(pos.max()) < 32, "instructions longer than 32 records"
    for c, m in ((2, 0xFFFFFFFF), (3, 0xFFFFFFFF), (1, 0x7F0000)):
        assert bool(((r[:, c] & m) == (r[hidx, c] & m)[iid]).all()), "non-uniform instruction"
    assert bool(((hi >> 24) == 0).all()), "reserved bits"
    I = hidx.shape[0]
    addr = torch.zeros((I, 32), dtype=torch.int64, device=dev)
    act = torch.zeros((I, 32), dtype=torch.bool, device=dev)
    addr[iid, pos] = ((hi & 0xFFFF) << 32) | r[:, 0]
    act[iid, pos] = True
    h = hi[hidx]
    flags = ((h >> 16) & 7) | (((h >> 19) & 3) << 3) | (((h >> 21) & 3) << 5)
    return pack_warp_records(addr, act, r[hidx, 2], r[hidx, 3], flags)


def instr_starts(records: torch.Tensor) -> torch.Tensor:
    """Indices of records whose instr_start bit is set (record 0 always starts)."""
    s = ((records[:, 1].to(torch.int64) >> 23) & 1).to(torch.bool)
    s[0] = True
    return torch.nonzero(s).flatten()


def shuffle_instructions(records: torch.Tensor, seed: int) -> torch.Tensor:
    """Seeded permutation of whole warp-instructions (SURVEY §8d variant)."""
    n = records.shape[0]
    starts = instr_starts(records).cpu()
    ends = torch.cat([starts[1:], torch.tensor([n])])
    g = torch.Generator().manual_seed(seed)
    perm = torch.randperm(len(starts), generator=g)
    idx = torch.cat([torch.arange(int(starts[p]), int(ends[p])) for p in perm.tolist()])
    return records[idx.to(records.device)]


def split_calls(n: int, records: torch.Tensor, n_calls: int) -> list:
    """Split into ~n_calls ingest calls, each beginning at an instr_start record."""
    starts = instr_starts(records).cpu().tolist()
    cuts = sorted({starts[min(len(starts) - 1, (i * len(starts)) // n_calls)] for i in range(n_calls)})
    cuts = [c for c in cuts if c > 0]
    bounds = [0] + cuts + [n]
    return [(bounds[i], bounds[i + 1]) for i in range(len(bounds) - 1) if bounds[i + 1] > bounds[i]]


# splitmix64 as a counter-based generator on int64 tensors (wrapping arithmetic)
def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser of (x + golden); int64 tensors, two's-complement wrap."""
    def c(v):
        return v - (1 << 64) if v >= (1 << 63) else v
    z = x.to(torch.int64) + c(0x9E3779B97F4A7C15)
    z = (z ^ _lsr(z, 30)) * c(0xBF58476D1CE4E5B9)
    z = (z ^ _lsr(z, 27)) * c(0x94D049BB133111EB)
    return z ^ _lsr(z, 31)


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical shift right of int64 bit patterns."""
    return (z >> k) & ((1 << (64 - k)) - 1)


from .workloads import (  # noqa: E402
    tiny, fig3, fig6, gemm, stencil, spmv, strided_gather, smem_thread_local,
    smem_warp_broadcast, random_trace, synthetic, random_warp_trace, hot_temps, hot_spots, WORKLOADS,
)

__all__ = [
    "Trace", "pack_records", "from_instructions", "shuffle_instructions", "split_calls",
    "pack_warp_records", "to_warp_records", "random_warp_trace",
    "instr_starts", "splitmix64", "tiny", "fig3", "fig6", "gemm", "stencil", "spmv",
    "strided_gather", "smem_thread_local", "smem_warp_broadcast", "random_trace",
    "synthetic", "hot_temps", "hot_spots", "WORKLOADS",
]
