#!/usr/bin/env python
"""bench.py -- trace records/s into the cuThermo heat map on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload sgemm]
                    [--impl ours|reference] [--dedup auto|sort|hash]

One step = one pass of the whole hot path over one
synthetic trace: thermo_reset + thermo_ingest_trace + thermo_build_heatmap +
thermo_classify, inputs resident in HBM.  The default workload is BJ
configs[1], the naive SGEMM 1024x1024 trace (K = 128: 270,532,608 records, G19).
Inputs (4.3 GB) are larger than L2 (126 MB), so no explicit flush is needed.

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle (the
reference arm of this tier) on bounded samples of the same workload.

Multi-GPU (torchrun, one process per GPU, NCCL): the sharded mode (row e) --
the workload grows with N (SGEMM with M = 1024 N: N x 270.5 M records, weak
scaling), each rank decodes its slice of warps, keys move to their sector's
owner in one all-to-all inside thermo_build_heatmap, and histograms/indicators
are combined by all-reduce; the step time is the max over ranks.
`--mode replicas` instead runs N independent copies (no exchange).
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
ALGO_BYTES = {  # 16 N + 16 U + 4 (words + sectors), per config
    "sgemm": dict(N=270532608, U=22020096, cells=9 * 163840),
}


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


def make_trace(workload: str, device: str, rank: int = 0, ws: int = 1):
    """The workload; with ws > 1 (sharded) rank's slice of the ws-times larger job."""
    import tracegen as tg
    if workload == "sgemm":
        if ws > 1:  # SGEMM with M = 1024 ws; rank r holds warps [r W / ws, (r + 1) W / ws)
            W = 32 * ws * 32 * 32
            return tg.gemm(1024 * ws, 1024, 128, "v00", device=device,
                           warp_range=(rank * W // ws, (rank + 1) * W // ws))
        return tg.gemm(1024, 1024, 128, "v00", device=device)
    if workload == "stencil":
        return tg.stencil(8192, device=device)
    if workload == "tiny":
        return tg.tiny("B", device=device)
    if workload == "spmv":
        return tg.spmv(24, 16, device=device)
    if workload == "synthetic":
        # BJ configs[4]: the 4-billion-record, 64-object, 8-launch job of 8 GPUs;
        # a rank holds 2^15 warps of every launch (2^29 records, 8.6 GB), so
        # ws ranks run the (ws/8)-scaled job and 8 ranks the full 2^32 records
        W = (1 << 15) * ws
        return tg.synthetic(warps_per_launch=W, warp_range=(rank * (1 << 15), (rank + 1) * (1 << 15)),
                            device=device)
    raise SystemExit(f"unknown workload {workload}")


def cpu_baseline(workload: str, budget_s: float = 12.0):
    """The oracle as it stands, single-threaded on a host core, on a bounded
    prefix sample of the same trace (records/s)."""
    import oracle
    import tracegen as tg
    if workload == "sgemm":   # a prefix of whole warps (the oracle runs ~2048 warps per 4 s)
        n_total = 270532608
        warps = max(64, int(2048 * budget_s / 4.0))
        t = tg.gemm(1024, 1024, 128, "v00", device="cpu", warp_limit=warps)
    else:
        t = make_trace(workload, "cpu")
        n_total = t.n
    recs = t.records
    o = oracle.Oracle([x[:4] for x in t.objects])
    chunk = 1 << 22
    done, t0 = 0, time.perf_counter()
    while done < recs.shape[0] and time.perf_counter() - t0 < 3 * budget_s:
        o.ingest(recs[done:done + chunk])
        done += min(chunk, recs.shape[0] - done)
    o.build()
    o.classify()
    el = time.perf_counter() - t0
    return {"value": done / el, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"first {done} of {n_total} records of the {workload} trace (ingest + build + classify, "
                      f"single-threaded std::set oracle, {el:.1f} s)"}


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
    n_total, n_obj = {"sgemm": (270532608, 3)}.get(args.workload, (None, None))
    restrict = None
    if args.workload == "sgemm":
        t = tg.gemm(1024, 1024, 128, "v00", device="cpu", warp_limit=1024)  # ~2 s of oracle work per step
    elif args.workload == "synthetic":
        # 32 warps of every launch (524,288 records); the oracle builds the rows
        # of the sectors they touch only (its sampled mode: every other row is 0)
        t = tg.synthetic(warps_per_launch=1 << 15, warp_range=(0, 32), device="cpu")
        n_total, n_obj = 1 << 29, len(t.objects)
        restrict = touched_sectors(t)
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
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": args.workload, "records": n_total, "objects": n_obj, "sample": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="sgemm")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dedup", default="auto", choices=["auto", "sort", "hash", "segment", "dense"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="sharded", choices=["sharded", "replicas"],
                    help="multi-GPU: one sharded job (default) or independent replicas")
    ap.add_argument("--format", default="lane", choices=["lane", "warp"],
                    help="record format: 16-B per-lane records (default, the contract) or 272-B "
                         "warp-instruction records (SURVEY §8f item 4)")
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
    from paper_2507_18729_b200 import BOTH, Thermo
    from paper_2507_18729_b200.thermo import nccl_unique_id
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = (ws > 1 or args.force_dist) and args.mode == "sharded"
    if args.force_dist:
        os.environ["THERMO_FORCE_COMM"] = "1"
    t = make_trace(args.workload, str(dev), rank, ws if sharded else 1)
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

    for _ in range(max(3, args.warmup)):
        step(inputs)
    st0 = th.stats()
    launches0 = st0["kernel_launches"]
    dec_ms, phase = [], {k: [] for k in ("ms_decode", "ms_dedup", "ms_count", "ms_hist", "ms_pc", "ms_indicators")}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step(inputs)
            s = th.stats()
            for k in phase:
                phase[k].append(s[k])
        e1.record(stream)
        barrier()
    ms_total = e0.elapsed_time(e1)
    ms = ms_total / args.steps
    launches = th.stats()["kernel_launches"] - launches0
    if ws > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = n * ws / (ms / 1e3)
    st = th.stats()
    clocks = clk.summary()

    # ---- e2e: same step through the C ABI with a pinned HOST trace ----
    e2e = None
    if not args.no_e2e:
        host = torch.empty_like(inputs, device="cpu").pin_memory()
        host.copy_(inputs)
        step(host)
        barrier()
        t0 = time.perf_counter()
        k2 = max(1, min(3, args.steps))
        for _ in range(k2):
            res = step(host)
        barrier()
        el = (time.perf_counter() - t0) / k2
        d2h = len(res) * 136
        e2e = {"value": n * ws / el, "unit": UNIT, "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": d2h,
               "ms_per_step": el * 1e3}
        del host

    # ---- roofline of the dominant kernel (decode: a2 + a3) ----
    peak, peak_kind = peaks()
    dec = statistics.mean(phase["ms_decode"])
    ph_mean = {k: statistics.mean(v) for k, v in phase.items()}
    dominant = max(ph_mean, key=ph_mean.get)
    achieved = in_bytes / (dec / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "decode_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(args.workload if args.format == "lane" else args.workload + "-warp")
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "kernel": "decode_kernel (a2+a3)" if args.format == "lane" else "decode_warp_kernel (a2+a3)",
            "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
            "algorithmic_bytes_per_launch": in_bytes, "ms_per_launch": dec}
    pipe = None
    if args.workload in ALGO_BYTES and ws == 1:
        a = ALGO_BYTES[args.workload]
        b = 16 * a["N"] + 16 * a["U"] + 4 * a["cells"]
        pipe = {"algorithmic_bytes": b, "achieved_GBps": b / (ms / 1e3) / 1e9,
                "frac": b / (ms / 1e3) / 1e9 / peak}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": args.workload, "records": n * ws, "format": args.format, "objects": len(t.objects),
                       "dedup": {1: "sort", 2: "hash", 3: "segment", 4: "dense"}.get(st["dedup_used"], "?"),
                       "l2": "inputs larger than L2 (16 B x records >> 126 MB), no flush",
                       "records_per_gpu": n, "parallelism": parallelism},
            "roofline": roof, "pipeline_roofline": pipe, "phase_ms": ph_mean, "dominant_phase": dominant,
            "clocks": clocks, "gpu_launches": launches,
            "stats": {k: st[k] for k in ("keys_emitted", "pc_keys_emitted", "distinct_pairs", "distinct_pc_pairs",
                                          "n_pcs")},
            "e2e": e2e}
    if sharded:  # NVLink roofline of the key all-to-all (row e), slowest rank
        xt = torch.tensor([st["ms_exchange"], float(st["exchange_bytes"])], device=dev, dtype=torch.float64)
        if ws > 1:
            dist.all_reduce(xt, op=dist.ReduceOp.MAX)
        xms, xb = float(xt[0]), float(xt[1])
        line["nvlink"] = {"exchange_ms": xms, "bytes_sent_per_rank": xb,
                          "achieved": xb / (xms / 1e3) / 1e9 if xms > 0 else None, "peak": 900.0, "unit": "GB/s",
                          "frac": (xb / (xms / 1e3) / 1e9) / 900.0 if xms > 0 else None}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and args.workload != "synthetic":
        line["cpu_baseline"] = cpu_baseline(args.workload)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
