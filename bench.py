#!/usr/bin/env python
"""bench.py -- trace records/s into the cuThermo heat map on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload spmv]
                    [--impl ours|reference] [--dedup auto|sort|hash|segment]

One step = one pass of the whole hot path over one
synthetic trace: thermo_reset + thermo_ingest_trace + thermo_build_heatmap +
thermo_classify, inputs resident in HBM (every trace is larger than the 126 MB
L2, so no explicit flush is needed).  The headline workload is BJ configs[3],
the CSR SpMV trace on an R-MAT scale-24 matrix (840.6 M records): the largest
single-GPU configuration and the one BJ's metric quotes at 1/2/4/8 B200.  The
default run also measures configs[1] (SGEMM), configs[2] (stencil) and
configs[4] (one rank's synthetic slice) and reports them under "configs".

Prints ONE JSON line (rank 0) with, per config, the dominant kernel's roofline
(algorithmic bytes per launch / its event-timed duration), the whole-pipeline
roofline (16 N + 16 U + 4 cells bytes), per-kernel times, and for
the headline the e2e rate through the C ABI from pinned host memory, the CPU
oracle baseline and the clocks of the timed region.  `--impl reference` times
the CPU oracle (the reference arm of this tier) on bounded samples.

Multi-GPU (torchrun, one process per GPU, NCCL): the sharded mode (row e).
SpMV: the same matrix split by rows over the ranks (strong scaling); SGEMM and
synthetic: each rank adds its own slice (weak scaling).  Keys move to their
sector's owner in one all-to-all inside thermo_build_heatmap; the step time is
the max over ranks.  `--mode replicas` instead runs N independent copies.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trace records/sec into heat map (1/2/4/8 B200) and achieved HBM GB/s vs peak"
UNIT = "records/s"
HEADLINE = "spmv"
OTHERS = ("sgemm", "stencil", "synthetic")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled during the timed region:
    NVML polled every 5 ms from a thread (nvidia-smi -lms 20 as the fallback).
    __enter__ returns only once the first sample has arrived, so the timed
    region that follows is covered; __exit__ keeps the samples taken up to the
    end of the region plus the first one after it."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc, self.stop = index, [], None, False
        self.t_start, self.t_end = 0.0, None

    def _nvml(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        bits = (pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

        def poll():
            try:
                while not self.stop:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((time.perf_counter(), float(sm), float(mx), tuple(bool(r & b) for b in bits)))
                    time.sleep(0.005)
            finally:
                pynvml.nvmlShutdown()
        return poll

    def _smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits", "-lms", "20"],
                                     stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

        def read():
            for line in self.proc.stdout:
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 6 and p[0].replace(".", "").isdigit():
                    self.rows.append((time.perf_counter(), float(p[0]),
                                      float(p[1]) if p[1].replace(".", "").isdigit() else float(p[0]),
                                      tuple(x.lower() == "active" for x in p[2:6])))
        return read

    def __enter__(self):
        try:
            target = self._nvml()
        except Exception:
            try:
                target = self._smi()
            except FileNotFoundError:
                return self
        self.t = threading.Thread(target=target, daemon=True)
        self.t.start()
        t0 = time.perf_counter()
        while not self.rows and time.perf_counter() - t0 < 10.0:
            time.sleep(0.005)
        self.t_start = time.perf_counter()
        return self

    def __exit__(self, *a):
        self.t_end = time.perf_counter()
        t0 = time.perf_counter()
        while not any(r[0] > self.t_end for r in self.rows) and time.perf_counter() - t0 < 2.0:
            time.sleep(0.005)
        self.stop = True
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        t0 = getattr(self, "t_start", 0.0)
        t1 = self.t_end if self.t_end is not None else float("inf")
        rows = [r for r in self.rows if t0 <= r[0] <= t1]
        if not rows:  # a region shorter than the sampling period: the samples around it
            rows = [r for r in self.rows if r[0] < t0][-1:] + [r for r in self.rows if r[0] > t1][:1]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({self.NAMES[i] for r in rows for i in range(4) if r[3][i]})
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def describe(workload: str, t) -> str:
    m = t.meta
    if workload == "spmv":
        return (f"CSR SpMV (Listing 5, one thread per row, block 256) on an R-MAT scale-{m['scale']} edge-factor-"
                f"{m['edgefactor']} matrix (Graph500 a,b,c,d = 0.57,0.19,0.19,0.05; {m['n']} rows, {m['nnz']} nnz)")
    if workload == "sgemm":
        return "naive SGEMM gemm_v00 (Listing 1), M = N = 1024, K = 128, block 32x32"
    if workload == "stencil":
        return "2-D 5-point stencil 8192^2, column-mapped (block 32x8), halo + uncoalesced column accesses"
    if workload == "synthetic":
        return "synthetic 64-object 8-launch trace, one rank's slice (2^15 warps per launch, 2^29 records)"
    return workload


def make_trace(workload: str, device: str, rank: int = 0, ws: int = 1):
    """The workload; with ws > 1 (sharded) rank's slice of the job."""
    import tracegen as tg
    if workload == "sgemm":
        if ws > 1:  # SGEMM with M = 1024 ws; rank r holds warps [r W / ws, (r + 1) W / ws)  (weak scaling)
            W = 32 * ws * 32 * 32
            return tg.gemm(1024 * ws, 1024, 128, "v00", device=device,
                           warp_range=(rank * W // ws, (rank + 1) * W // ws))
        return tg.gemm(1024, 1024, 128, "v00", device=device)
    if workload == "stencil":
        return tg.stencil(8192, device=device)
    if workload == "tiny":
        return tg.tiny("B", device=device)
    if workload == "spmv":
        # the same scale-24 matrix for every N (strong scaling): rank r holds
        # the rows [r n / ws, (r + 1) n / ws) (whole warps)
        n = 1 << 24
        lo, hi = (rank * n // ws) // 32 * 32, ((rank + 1) * n // ws) // 32 * 32
        return tg.spmv(24, 16, device=device, row_range=(lo, hi) if ws > 1 else None)
    if workload == "synthetic":
        # BJ configs[4]: the 4-billion-record, 64-object, 8-launch job of 8 GPUs;
        # a rank holds 2^15 warps of every launch (2^29 records, 8.6 GB), so
        # ws ranks run the (ws/8)-scaled job and 8 ranks the full 2^32 records
        W = (1 << 15) * ws
        return tg.synthetic(warps_per_launch=W, warp_range=(rank * (1 << 15), (rank + 1) * (1 << 15)),
                            device=device)
    raise SystemExit(f"unknown workload {workload}")


def host_info():
    model = "?"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def cpu_baseline(workload: str, t=None, budget_s: float = 12.0):
    """The oracle as it stands, single-threaded on one host core, on a bounded
    prefix sample of the same trace (records/s): ingest + build + classify."""
    import oracle
    import tracegen as tg
    if workload == "sgemm":   # a prefix of whole warps (the oracle runs ~2048 warps per 4 s)
        n_total = 270532608
        warps = max(64, int(2048 * budget_s / 4.0))
        tt = tg.gemm(1024, 1024, 128, "v00", device="cpu", warp_limit=warps)
        objects, recs = tt.objects, tt.records
    else:
        n_total = t.n
        k = min(t.n, 4_000_000)  # a prefix of the trace (whole source warps; the reference arm's sample)
        objects, recs = t.objects, t.records[:k].cpu()
    o = oracle.Oracle([x[:4] for x in objects])
    chunk = 1 << 20
    done, t0 = 0, time.perf_counter()
    while done < recs.shape[0] and time.perf_counter() - t0 < budget_s:
        o.ingest(recs[done:done + chunk])
        done += min(chunk, recs.shape[0] - done)
    o.build()
    o.classify()
    el = time.perf_counter() - t0
    return {"value": done / el, "unit": UNIT, "cores": 1, "kind": "oracle", **host_info(),
            "sample": f"first {done} of {n_total} records of the {workload} trace (ingest + build + classify, "
                      f"single-threaded std::set oracle, {el:.1f} s)"}


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    return ws, rank, local


def run_reference(args, ws, rank):
    """The reference arm of this tier: the CPU oracle as it stands, single-threaded,
    each step a bounded sample (a prefix of whole warps) of the same workload."""
    if rank != 0:
        return
    import oracle
    import tracegen as tg
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"  # input generation only
    restrict = None
    if args.workload == "sgemm":
        t = tg.gemm(1024, 1024, 128, "v00", device="cpu", warp_limit=1024)  # ~2 s of oracle work per step
        n_total, n_obj = 270532608, 3
    elif args.workload == "synthetic":
        # 32 warps of every launch (524,288 records); the oracle builds the rows
        # of the sectors they touch only (its sampled mode: every other row is 0)
        t = tg.synthetic(warps_per_launch=1 << 15, warp_range=(0, 32), device="cpu")
        n_total, n_obj = 1 << 29, len(t.objects)
        restrict = touched_sectors(t)
    elif args.workload in ("spmv", "stencil"):
        full = make_trace(args.workload, dev)
        n_total, n_obj = full.n, len(full.objects)
        k = 4_000_000  # the first 4 M records (whole source warps: ~2 s of oracle work per step)
        t = tg.Trace(full.name, full.objects, full.records[:k].cpu().clone(), meta=full.meta)
        del full
    else:
        t = make_trace(args.workload, "cpu")
        n_total, n_obj = t.n, len(t.objects)

    def step():
        o = oracle.Oracle([x[:4] for x in t.objects])
        if restrict is not None:
            o.restrict(*restrict)
        o.ingest(t.records)
        o.build()
        o.classify()

    for _ in range(max(3, args.warmup)):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    v = t.n * args.steps / el
    sample = (f"first {t.n} of {n_total} records of the {args.workload} trace per step (ingest + build + "
              f"classify, single-threaded std::set oracle)")
    if restrict is not None:
        sample = (f"warps 0-31 of every launch: {t.n} of the {n_total} records of one rank's synthetic slice per "
                  f"step (ingest + build of the {len(restrict[0])} sectors they touch, oracle sampled mode; "
                  f"single-threaded std::set oracle)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong" if args.workload == "spmv" else "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": args.workload, "records": n_total, "objects": n_obj, "sample": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             **host_info()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def touched_sectors(t):
    """(object index, local sector) of every sector a record touches (plain
    numpy over the record fields; the oracle's sampled mode is given these)."""
    import numpy as np
    r = t.records.numpy().view(np.uint32)
    addr = r[:, 0].astype(np.uint64) | ((r[:, 1].astype(np.uint64) & 0xFFFF) << np.uint64(32))
    size = np.left_shift(np.uint64(1), (r[:, 1].astype(np.uint64) >> np.uint64(16)) & np.uint64(7))
    sec = np.unique(np.concatenate([addr >> np.uint64(5), (addr + size - np.uint64(1)) >> np.uint64(5)]))
    bases = np.array([o[0] for o in t.objects], dtype=np.uint64)
    lens = np.array([o[1] for o in t.objects], dtype=np.uint64)
    order = np.argsort(bases)
    k = np.searchsorted(bases[order], sec << np.uint64(5), side="right") - 1
    ok = k >= 0
    oi = order[np.where(ok, k, 0)]
    ok &= (sec << np.uint64(5)) < bases[oi] + lens[oi]
    return oi[ok].astype(np.uint32), (sec[ok] - bases[oi[ok]] // np.uint64(32)).astype(np.uint64)


# algorithmic bytes per launch of each kernel:
#   decode_kernel       16 B per record (the trace, read once); the same for
#                       decode_lane_kernel (the lane-per-record decoder)
#   seg_coarse_kernel   16 B per key (read + write)          [partition pass 1]
#   seg_fine_kernel     16 B per key (read + write)          [partition pass 2]
#   seg_chunk_kernel     8 B per key (read once) + 36 B per touched sector (its row written)
#   object_hist_kernel  36 B per registered sector (the dense rows, read once)
#   indicator_kernels   72 B per registered sector (two tile passes over the rows)
# (decode_general_kernel, seg_scan and seg_big_kernel re-read subsets whose
# sizes the library does not report; they are listed with their times only)
def kernel_bytes(k, n, st, S_tot, touched):
    keys = st["keys_emitted"]
    return {"decode_kernel": 16 * n, "decode_lane_kernel": 16 * n, "seg_coarse_kernel": 16 * keys, "seg_fine_kernel": 16 * keys,
            "seg_chunk_kernel": 8 * keys + 36 * touched, "object_hist_kernel": 36 * S_tot,
            "indicator_kernels": 72 * S_tot}.get(k)


def load_traffic():
    p = os.path.join(ROOT, "profiles", "r2_traffic.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


def run_ours(args, workload, ws, rank, local, steps, warmup, headline):
    import torch
    import torch.distributed as dist
    from paper_2507_18729_b200 import BOTH, Thermo
    from paper_2507_18729_b200.thermo import nccl_unique_id
    dev = torch.device("cuda", local)
    sharded = (ws > 1 or args.force_dist) and args.mode == "sharded"
    t = make_trace(workload, str(dev), rank, ws if sharded else 1)
    n = t.n
    stream = torch.cuda.current_stream(dev)
    dedup = {"auto": 0, "sort": 1, "hash": 2, "segment": 3, "dense": 4}[args.dedup]
    cfg = dict(max_launches=max(1, int(t.meta.get("launches", 1))),
               max_warps_per_launch=max(1, int(t.meta.get("warps", 1 << 20))),
               max_pcs=int(t.meta.get("pcs", 256)), dedup=dedup)
    parallelism = "single"
    if sharded:
        from paper_2507_18729_b200.dist import broadcast_bytes
        uid = broadcast_bytes(nccl_unique_id() if rank == 0 else None) if ws > 1 else nccl_unique_id()
        th = Thermo.dist(uid, rank, ws, device=local, stream=stream.cuda_stream, **cfg)
        parallelism = f"sharded x{ws}: sector owners, one NCCL all-to-all of keys + all-reduce of sums"
    else:
        th = Thermo(device=local, stream=stream.cuda_stream, **cfg)
        if ws > 1:
            parallelism = f"replicas x{ws}"
    th.register_objects(t.objects)
    S_tot = sum((o[1] + 31) // 32 for o in t.objects)

    ingest = th.ingest
    inputs = t.records
    if args.format == "warp":  # warp-instruction records of the same trace
        import tracegen as tg
        inputs = tg.to_warp_records(t.records)
        t.records = None
        torch.cuda.empty_cache()
        ingest = th.ingest_warp
    in_bytes = inputs.numel() * 4

    def step(recs):
        th.reset()
        ingest(recs)
        th.build(BOTH)
        return th.classify()

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(3, warmup)):
        res = step(inputs)
    st0 = th.stats()
    launches0 = st0["kernel_launches"]
    phase = {k: [] for k in ("ms_decode", "ms_dedup", "ms_count", "ms_hist", "ms_pc", "ms_indicators")}
    kern = {k: [] for k in st0["ms_kernel"]}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(steps):
            res = step(inputs)
            s = th.stats()
            for k in phase:
                phase[k].append(s[k])
            for k in kern:
                kern[k].append(s["ms_kernel"][k])
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1) / steps
    launches = th.stats()["kernel_launches"] - launches0
    if ws > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    st = th.stats()
    n_job = n
    if ws > 1:  # records of the whole job (the ranks' slices differ for SpMV)
        nt = torch.tensor([n], device=dev, dtype=torch.int64)
        dist.all_reduce(nt)
        n_job = int(nt.item())
    value = n_job / (ms / 1e3)
    touched = sum(r["touched_sectors"] for r in res)

    peak, peak_kind = peaks()
    ph_mean = {k: statistics.mean(v) for k, v in phase.items()}
    k_mean = {k: statistics.mean(v) for k, v in kern.items()}
    traffic_db = load_traffic().get(workload if args.format == "lane" else workload + "-warp", {})
    kernels = {}
    # the decode timer covers whichever decoder the ingest chose (stats.decoder_used)
    dec_name = {2: "decode_lane_kernel", 3: "decode_warp_kernel"}.get(st.get("decoder_used", 1), "decode_kernel")
    for k, v in k_mean.items():
        if v <= 0:
            continue
        if k == "decode_kernel":
            k = dec_name
        b = kernel_bytes(k, n, st, S_tot, touched)
        if k in ("decode_kernel", "decode_warp_kernel") and args.format == "warp":
            b = in_bytes
        e = {"ms_per_launch": v}
        if b is not None:
            e.update(algorithmic_bytes_per_launch=b, achieved_GBps=b / (v / 1e3) / 1e9,
                     frac=b / (v / 1e3) / 1e9 / peak)
        kernels[k] = e
    # dominant kernel with an algorithmic byte count: the roofline line
    cand = [k for k in kernels if "algorithmic_bytes_per_launch" in kernels[k]]
    dom = max(cand, key=lambda k: kernels[k]["ms_per_launch"]) if cand else None
    roof = None
    if dom:
        d = kernels[dom]
        roof = {"bound": "hbm", "kernel": dom + (" (warp-instruction records)" if args.format == "warp" else ""),
                "achieved": d["achieved_GBps"], "peak": peak, "unit": "GB/s", "frac": d["frac"],
                "traffic": traffic_db.get(dom), "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": d["algorithmic_bytes_per_launch"], "ms_per_launch": d["ms_per_launch"],
                "share_of_step": d["ms_per_launch"] / ms}
    U = st["distinct_pairs"]
    b_pipe = 16 * n + 16 * U + 4 * 9 * S_tot
    pipe = {"algorithmic_bytes": b_pipe, "achieved_GBps": b_pipe / (ms / 1e3) / 1e9,
            "frac": b_pipe / (ms / 1e3) / 1e9 / peak, "N": n, "U": U, "cells": 9 * S_tot} if ws == 1 else None
    line = {"workload": workload, "value": value, "ms_per_step": ms, "records": n_job, "steps": steps,
            "description": describe(workload, t), "roofline": roof, "pipeline_roofline": pipe, "kernels": kernels,
            "phase_ms": ph_mean, "gpu_launches": launches,
            "stats": {k: st[k] for k in ("keys_emitted", "distinct_pairs", "distinct_pc_pairs", "n_pcs")},
            "dedup": {1: "sort", 2: "hash", 3: "segment", 4: "dense"}.get(st["dedup_used"], "?"),
            "parallelism": parallelism, "scaling": "strong" if workload == "spmv" else "weak"}
    if headline:
        line["clocks"] = clk.summary()
        # ---- e2e: same step through the C ABI with a pinned HOST trace ----
        if not args.no_e2e:
            host = torch.empty_like(inputs, device="cpu").pin_memory()
            host.copy_(inputs)
            step(host)
            barrier()
            t0 = time.perf_counter()
            k2 = max(1, min(3, steps))
            for _ in range(k2):
                r2 = step(host)
            barrier()
            el = (time.perf_counter() - t0) / k2
            line["e2e"] = {"value": n_job / el, "unit": UNIT, "h2d_bytes_per_step": in_bytes,
                           "d2h_bytes_per_step": len(r2) * 136, "ms_per_step": el * 1e3}
            del host
        if sharded:  # NVLink roofline of the key all-to-all (row e), slowest rank
            xt = torch.tensor([st["ms_exchange"], float(st["exchange_bytes"])], device=dev, dtype=torch.float64)
            if ws > 1:
                dist.all_reduce(xt, op=dist.ReduceOp.MAX)
            xms, xb = float(xt[0]), float(xt[1])
            line["nvlink"] = {"exchange_ms": xms, "bytes_sent_per_rank": xb,
                              "achieved": xb / (xms / 1e3) / 1e9 if xms > 0 else None, "peak": 900.0, "unit": "GB/s",
                              "frac": (xb / (xms / 1e3) / 1e9) / 900.0 if xms > 0 else None}
        if rank == 0 and ws == 1 and not args.no_cpu_baseline and workload != "synthetic":
            line["cpu_baseline"] = cpu_baseline(workload, t)
    th.close()
    del th, inputs, t
    torch.cuda.empty_cache()
    return line


def run_local_shards(args, P):
    """P in-process shards of the sharded mode on one GPU (thermo_create_local_shards,
    the same exchange algorithm as the NCCL ranks, device-to-device copies):
    the trace split at instruction heads into P slices, one host thread per
    rank.  Reports, per rank, the sectors its dense rows cover (storage falls
    as 1/P by construction), the keys it counts after the exchange, the bytes
    it sends, and its device times per phase; the ranks share one GPU, so the
    times show the per-rank work, not a multi-GPU speed-up."""
    import torch
    from paper_2507_18729_b200 import BOTH, Thermo
    from paper_2507_18729_b200.dist import run_ranks, split_at_heads
    t = make_trace(args.workload, "cuda")
    cfg = dict(max_launches=max(1, int(t.meta.get("launches", 1))),
               max_warps_per_launch=max(1, int(t.meta.get("warps", 1 << 20))), max_pcs=int(t.meta.get("pcs", 256)))
    cuts = split_at_heads(t.records, P)
    slices = [t.records[a:b] for a, b in cuts]
    shards = Thermo.local_shards(P, **cfg) if P > 1 else [Thermo(**cfg)]
    for th in shards:
        th.register_objects(t.objects)

    def step(r):
        def f():
            th = shards[r]
            th.reset()
            if slices[r].shape[0]:
                th.ingest(slices[r])
            th.build(BOTH)
            th.classify()
            return th.stats()
        return f

    for _ in range(max(1, args.warmup)):
        run_ranks([step(r) for r in range(P)])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sts = run_ranks([step(r) for r in range(P)])
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) / args.steps
    ranks = [{"rank": r, "records": int(slices[r].shape[0]), "local_sectors": st["local_sectors"],
              "dense_row_bytes": 36 * st["local_sectors"], "keys_counted": st["local_keys"],
              "exchange_bytes_sent": st["exchange_bytes"], "ms_ingest": st["ms_ingest"], "ms_build": st["ms_build"],
              "ms_classify": st["ms_classify"], "ms_exchange": st["ms_exchange"],
              "ms_kernel": {k: v for k, v in st["ms_kernel"].items() if v > 0}} for r, st in enumerate(sts)]
    S_tot = sum((o[1] + 31) // 32 for o in t.objects)
    print(json.dumps({"mode": "local_shards", "workload": args.workload, "P": P, "records": t.n, "S_tot": S_tot,
                      "wall_ms_per_step": el * 1e3, "ranks": ranks}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=HEADLINE)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dedup", default="auto", choices=["auto", "sort", "hash", "segment", "dense"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--only", action="store_true", help="measure the --workload config only (no 'configs')")
    ap.add_argument("--other-steps", type=int, default=5, help="timed steps of each non-headline config")
    ap.add_argument("--mode", default="sharded", choices=["sharded", "replicas"],
                    help="multi-GPU: one sharded job (default) or independent replicas")
    ap.add_argument("--format", default="lane", choices=["lane", "warp"],
                    help="record format: 16-B per-lane records (default, the contract) or 272-B "
                         "warp-instruction records (SURVEY §8f item 4)")
    ap.add_argument("--local-shards", type=int, default=0,
                    help="P in-process shards on one GPU: per-rank storage, keys and phase times (no bench line)")
    ap.add_argument("--force-dist", action="store_true",
                    help="one GPU through the sharded NCCL path (checks that code path on one GPU)")
    args = ap.parse_args()
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if args.local_shards:
        run_local_shards(args, args.local_shards)
        return
    if args.force_dist:
        os.environ["THERMO_FORCE_COMM"] = "1"
    h = run_ours(args, args.workload, ws, rank, local, args.steps, args.warmup, True)
    others = {}
    if not args.only and ws == 1 and args.workload == HEADLINE and args.format == "lane":
        for w in OTHERS:
            others[w] = run_ours(args, w, ws, rank, local, args.other_steps, args.warmup, False)
    line = {"metric": METRIC, "value": h["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": h["ms_per_step"], "higher_is_better": True,
            "scaling": h["scaling"], "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": args.workload, "description": h["description"], "records": h["records"],
                       "records_per_gpu": h["records"] // ws if ws else h["records"], "format": args.format,
                       "dedup": h["dedup"], "parallelism": h["parallelism"],
                       "l2": "inputs larger than L2 (16 B x records >> 126 MB), no flush"},
            "roofline": h["roofline"], "pipeline_roofline": h["pipeline_roofline"], "kernels": h["kernels"],
            "phase_ms": h["phase_ms"], "clocks": h.get("clocks"), "gpu_launches": h["gpu_launches"],
            "stats": h["stats"], "e2e": h.get("e2e")}
    for k in ("nvlink", "cpu_baseline"):
        if k in h:
            line[k] = h[k]
    if others:
        line["configs"] = others
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
