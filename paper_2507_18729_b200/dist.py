"""Host-side plumbing of the address-sharded mode (row e).

The reduction itself -- pc-id unification, the key all-to-all to sector
owners, the per-owner counts and the combination of histograms and indicator
sums -- runs inside libthermo (csrc/shard.cu, NCCL over NVLink).  This module
only does what sits around it on the host:

* split a trace into per-rank slices at instruction heads (each ingest call
  starts an instruction, G24, so a slice must begin at an instr_start record);
* hand rank 0's ncclUniqueId to the other ranks over a torch.distributed group;
* assemble full heat-map rows from the ranks' partitions (cells of sectors a
  rank does not own are 0, so the rows are the element-wise sum);
* drive the in-process shards (thermo_create_local_shards) from one thread each.
"""
from __future__ import annotations

import threading

import numpy as np

INSTR_START_BIT = 23  # bit 55 of addr_flags = bit 23 of the record's second int32


def split_at_heads(records, nparts: int) -> list[tuple[int, int]]:
    """[start, end) slices of about len/nparts records each, every slice but the
    first starting at an instr_start record.  records: int32 [n, 4] (torch or
    numpy, any device).  Slices may be empty when heads are sparse."""
    n = int(records.shape[0])
    if nparts <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(0, nparts - 1)
    col = records[:, 1]
    if hasattr(col, "cpu"):
        col = col.cpu().numpy()
    heads = np.flatnonzero((np.asarray(col).astype(np.int64) >> INSTR_START_BIT) & 1)
    cuts = [0]
    for r in range(1, nparts):
        target = (n * r) // nparts
        i = int(np.searchsorted(heads, target))
        c = int(heads[i]) if i < len(heads) else n
        cuts.append(max(c, cuts[-1]))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(nparts)]


def broadcast_bytes(payload: bytes | None, src: int = 0, group=None) -> bytes:
    """Broadcast a small byte string (e.g. the 128-byte ncclUniqueId) from src."""
    import torch.distributed as dist

    obj = [payload if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def assemble_rows(part: np.ndarray, group=None, device=None) -> np.ndarray:
    """Full heat-map rows from this rank's partition: element-wise sum over ranks."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.asarray(part).astype(np.int64))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy().astype(part.dtype)


def run_ranks(fns) -> list:
    """Run fns[r]() on one thread per rank (the collective calls of in-process
    shards block until every rank arrives); returns their results, re-raising
    the first exception."""
    out = [None] * len(fns)
    err = [None] * len(fns)

    def body(r):
        try:
            out[r] = fns[r]()
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out
