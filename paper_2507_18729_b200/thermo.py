"""Thin ctypes binding of libthermo (include/thermo.h).

Argument marshalling only: every step of the heat-map reduction runs in the
library's sm_100a kernels.  There is no CPU fallback -- if libthermo.so is
missing or no CUDA device is visible, the calls raise.

Low-level names mirror the C ABI (``thermo_create``, ``thermo_register_objects``,
``thermo_ingest_trace``, ``thermo_build_heatmap``, ``thermo_query_heatmap``,
``thermo_query_histogram``, ``thermo_query_per_pc``, ``thermo_classify``,
``thermo_get_stats``); ``Thermo`` wraps one context.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libthermo.so")

WORD, SECTOR, BOTH = 1, 2, 3
DEDUP_AUTO, DEDUP_SORT, DEDUP_HASH, DEDUP_SEGMENT, DEDUP_DENSE = 0, 1, 2, 3, 4
ALL_LAUNCHES = 0xFFFFFFFF
LEVELS = 33
STATUS = {0: "OK", -1: "EINVAL", -2: "ENOMEM", -3: "ERANGE", -4: "ESTATE", -5: "ECUDA", -6: "ENCCL"}
LABELS = {"Hot": 1, "RandomHot": 2, "FalseSharing": 4, "SmemAbuseThreadLocal": 8,
          "SmemAbuseWarpPrivate": 16, "Misaligned": 32, "Strided": 64}

u32, u64, vp, sz = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t


class thermo_object(ctypes.Structure):
    _fields_ = [("base", u64), ("len", u64), ("space", u32), ("id", u32)]


class thermo_config(ctypes.Structure):
    _fields_ = [("max_launches", u32), ("max_warps_per_launch", u32), ("max_pcs", u32), ("dedup", u32),
                ("track_pc", u32), ("track_access", u32), ("expected_pairs", u64),
                ("block_warps", u32), ("block_id", u32)]


PARAM_FIELDS = ("theta_hot", "alpha_num", "alpha_den", "beta_num", "beta_den", "fs_min", "smem_cap",
                "smem_cov_num", "smem_cov_den", "gamma_num", "gamma_den", "strided_min_sectors", "dom_num",
                "dom_den", "hot_frac_num", "hot_frac_den", "fs_frac_num", "fs_frac_den", "mis_frac_num",
                "mis_frac_den", "cv_num", "cv_den")


class thermo_params(ctypes.Structure):
    _fields_ = [(f, u64) for f in PARAM_FIELDS]


IND_FIELDS = ("n_words", "n_sectors", "touched_sectors", "touched_words", "hot_sectors", "fs_sectors", "sum_x",
              "sum_x2_lo", "sum_x2_hi", "le1_words", "max_sector_count", "instrs", "misaligned_instrs", "gaps",
              "dom_gap", "dom_count")


class thermo_indicators(ctypes.Structure):
    _fields_ = [("object_id", u32), ("labels", u32)] + [(f, u64) for f in IND_FIELDS]


class thermo_pc_hist(ctypes.Structure):
    _fields_ = [("launch", u32), ("pc", u32), ("hist", u64 * LEVELS)]


class thermo_stats(ctypes.Structure):
    _fields_ = [("records", u64), ("invalid", u64), ("out_of_range", u64), ("unmapped_words", u64),
                ("mapped_word_accesses", u64), ("keys_emitted", u64), ("pc_keys_emitted", u64),
                ("distinct_pairs", u64), ("distinct_pc_pairs", u64), ("n_pcs", u64), ("dedup_used", u32), ("decoder_used", u32),
                ("ms_ingest", ctypes.c_double), ("ms_build", ctypes.c_double),
                ("ms_classify", ctypes.c_double), ("ms_decode", ctypes.c_double), ("ms_dedup", ctypes.c_double),
                ("ms_count", ctypes.c_double), ("ms_hist", ctypes.c_double), ("ms_pc", ctypes.c_double),
                ("ms_indicators", ctypes.c_double), ("kernel_launches", u64),
                ("ms_exchange", ctypes.c_double), ("exchange_bytes", u64), ("ms_kernel", ctypes.c_double * 9), ("local_sectors", u64), ("local_keys", u64)]


# every symbol include/thermo.h declares
EXPORTS = ("thermo_default_config", "thermo_default_params", "thermo_abi_version", "thermo_create",
           "thermo_create_dist", "thermo_nccl_unique_id", "thermo_destroy", "thermo_reset",
           "thermo_register_objects", "thermo_ingest_trace", "thermo_build_heatmap", "thermo_query_heatmap",
           "thermo_query_histogram", "thermo_query_per_pc", "thermo_classify", "thermo_get_stats",
           "thermo_last_error", "thermo_create_local_shards", "thermo_sharding", "thermo_query_access",
           "thermo_ingest_warp_trace", "thermo_query_runs", "thermo_set_launch_whitelist")

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libthermo.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -m paper_2507_18729_b200.build`")
    L = ctypes.CDLL(path)
    P = ctypes.POINTER
    L.thermo_default_config.argtypes = [P(thermo_config)]
    L.thermo_default_config.restype = None
    L.thermo_default_params.argtypes = [P(thermo_params)]
    L.thermo_default_params.restype = None
    L.thermo_abi_version.restype = u32
    L.thermo_create.argtypes = [P(vp), ctypes.c_int, vp, P(thermo_config)]
    L.thermo_create_dist.argtypes = [P(vp), ctypes.c_int, vp, P(thermo_config), vp, ctypes.c_int, ctypes.c_int]
    L.thermo_nccl_unique_id.argtypes = [vp]
    L.thermo_create_local_shards.argtypes = [P(vp), ctypes.c_int, P(thermo_config), ctypes.c_int]
    L.thermo_sharding.argtypes = [vp, P(ctypes.c_int), P(ctypes.c_int), P(u32)]
    L.thermo_destroy.argtypes = [vp]
    L.thermo_reset.argtypes = [vp]
    L.thermo_set_launch_whitelist.argtypes = [vp, vp, sz]
    L.thermo_register_objects.argtypes = [vp, P(thermo_object), sz]
    L.thermo_ingest_trace.argtypes = [vp, vp, sz]
    L.thermo_ingest_warp_trace.argtypes = [vp, vp, sz]
    L.thermo_build_heatmap.argtypes = [vp, ctypes.c_int, u32]
    L.thermo_query_heatmap.argtypes = [vp, u32, ctypes.c_int, vp, sz, P(sz)]
    L.thermo_query_histogram.argtypes = [vp, u32, ctypes.c_int, vp]
    L.thermo_query_access.argtypes = [vp, u32, vp, sz, P(sz)]
    L.thermo_query_runs.argtypes = [vp, u32, vp, sz, P(sz)]
    L.thermo_query_per_pc.argtypes = [vp, ctypes.c_int, P(thermo_pc_hist), sz, P(sz)]
    L.thermo_classify.argtypes = [vp, P(thermo_params), P(thermo_indicators), sz, P(sz)]
    L.thermo_get_stats.argtypes = [vp, P(thermo_stats)]
    L.thermo_last_error.argtypes = [vp]
    L.thermo_last_error.restype = ctypes.c_char_p
    for name in EXPORTS:
        if name not in ("thermo_default_config", "thermo_default_params", "thermo_abi_version",
                        "thermo_last_error"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


class ThermoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libthermo {STATUS.get(status, status)}: {msg}")
        self.status = status


def default_params() -> dict:
    p = thermo_params()
    load().thermo_default_params(ctypes.byref(p))
    return {f: getattr(p, f) for f in PARAM_FIELDS}


def label_names(bits: int) -> list[str]:
    return [k for k, v in LABELS.items() if bits & v]


def _config(max_launches: int = 1, max_warps_per_launch: int = 1 << 20, max_pcs: int = 4096,
            dedup: int = DEDUP_AUTO, track_pc: bool = True, track_access: bool = False, block_warps: int = 0,
            block_id: int = 0) -> thermo_config:
    cfg = thermo_config()
    load().thermo_default_config(ctypes.byref(cfg))
    cfg.max_launches, cfg.max_warps_per_launch, cfg.max_pcs = max_launches, max_warps_per_launch, max_pcs
    cfg.dedup, cfg.track_pc, cfg.track_access = dedup, int(bool(track_pc)), int(bool(track_access))
    cfg.block_warps, cfg.block_id = block_warps, block_id  # sampled-block mode (0: whole grid)
    return cfg


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (thermo_nccl_unique_id), made on rank 0."""
    buf = ctypes.create_string_buffer(128)
    st = load().thermo_nccl_unique_id(buf)
    if st:
        raise ThermoError(st, "thermo_nccl_unique_id")
    return buf.raw


# thermo_stats.ms_kernel entries (include/thermo.h THERMO_K_*)
KERNELS = ("decode_kernel", "decode_general_kernel", "seg_scan", "seg_coarse_kernel", "seg_fine_kernel",
           "seg_chunk_kernel", "seg_big_kernel", "object_hist_kernel", "indicator_kernels")


def _default_stream(device: int) -> int:
    """torch's current stream on `device` (records made by torch are ordered
    before the ingest that reads them).  0 for the legacy default stream: the
    library's own stream is then a blocking one, ordered after it as well."""
    try:
        import torch
        if torch.cuda.is_available():
            return int(torch.cuda.current_stream(device).cuda_stream)
    except Exception:
        pass
    return 0


class Thermo:
    """One libthermo context (bound to a CUDA device and stream).

    Records are int32 [n, 4] torch tensors (16-byte thermo_record) on the GPU
    (fast path) or in host memory (staged by the library).
    """

    def __init__(self, device: int = 0, stream=None, _handle=None, **cfg_kw):
        self.L = load()
        self.objects = []
        if _handle is not None:
            self.h = _handle
            return
        cfg = _config(**cfg_kw)
        h = vp()
        stream = _default_stream(device) if stream is None else stream
        st = self.L.thermo_create(ctypes.byref(h), device, vp(stream) if stream else None, ctypes.byref(cfg))
        if st:
            raise ThermoError(st, "thermo_create")
        self.h = h

    @classmethod
    def dist(cls, nccl_id: bytes, rank: int, nranks: int, device: int = 0, stream=None, **cfg_kw) -> "Thermo":
        """Rank `rank` of the address-sharded mode (thermo_create_dist): build and
        classify are collective; queries are job-wide except heatmap (this rank's
        partition, other ranks' sectors 0)."""
        L = load()
        cfg = _config(**cfg_kw)
        h = vp()
        stream = _default_stream(device) if stream is None else stream
        idb = ctypes.create_string_buffer(bytes(nccl_id), 128)
        st = L.thermo_create_dist(ctypes.byref(h), device, vp(stream) if stream else None, ctypes.byref(cfg), idb,
                                  rank, nranks)
        if st:
            raise ThermoError(st, "thermo_create_dist")
        return cls(_handle=h)

    @classmethod
    def local_shards(cls, nranks: int, device: int = 0, **cfg_kw) -> list:
        """nranks contexts of the sharded mode inside this process
        (thermo_create_local_shards); drive each from its own thread."""
        L = load()
        cfg = _config(**cfg_kw)
        hs = (vp * nranks)()
        st = L.thermo_create_local_shards(hs, device, ctypes.byref(cfg), nranks)
        if st:
            raise ThermoError(st, "thermo_create_local_shards")
        return [cls(_handle=vp(hs[r])) for r in range(nranks)]

    def sharding(self) -> tuple:
        """(rank, nranks, ownership chunk in sectors)."""
        r, n, c = ctypes.c_int(), ctypes.c_int(), u32()
        self._ck(self.L.thermo_sharding(self.h, ctypes.byref(r), ctypes.byref(n), ctypes.byref(c)))
        return r.value, n.value, c.value

    # ---- plumbing ----
    def _ck(self, st):
        if st:
            raise ThermoError(st, (self.L.thermo_last_error(self.h) or b"").decode())

    def close(self):
        if getattr(self, "h", None):
            self.L.thermo_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- the ABI ----
    def register_objects(self, objects):
        """objects: iterable of (base, len, space, id[, label])."""
        self.objects = [tuple(int(x) for x in o[:4]) for o in objects]
        arr = (thermo_object * len(self.objects))(*[thermo_object(*o) for o in self.objects])
        self._ck(self.L.thermo_register_objects(self.h, arr, len(self.objects)))

    def reset(self):
        self._ck(self.L.thermo_reset(self.h))

    def set_launch_whitelist(self, launches=()):
        """Kernel sampling by whitelist: only these launch ids are traced
        from the next ingest on; () traces every launch."""
        a = (ctypes.c_uint32 * max(1, len(launches)))(*[int(x) for x in launches])
        self._ck(self.L.thermo_set_launch_whitelist(self.h, ctypes.cast(a, ctypes.c_void_p) if launches else None,
                                                    len(launches)))

    def ingest(self, records):
        """records: torch int32 [n, 4] (device or host) or a numpy array."""
        if hasattr(records, "data_ptr"):
            assert records.is_contiguous() and records.element_size() * records.shape[-1] == 16
            ptr, n = records.data_ptr(), records.shape[0]
        else:
            a = np.ascontiguousarray(records)
            ptr, n = a.ctypes.data, a.nbytes // 16
            self._keep = a
        self._ck(self.L.thermo_ingest_trace(self.h, vp(ptr), n))

    def ingest_warp(self, records):
        """Warp-instruction records: torch int32 [n, 68] (272-byte thermo_warp_record), device or host."""
        assert records.is_contiguous() and records.shape[-1] == 68 and records.dtype.itemsize == 4
        self._ck(self.L.thermo_ingest_warp_trace(self.h, vp(records.data_ptr()), records.shape[0]))

    def ingest_ptr(self, ptr: int, n: int):
        self._ck(self.L.thermo_ingest_trace(self.h, vp(ptr), n))

    def build(self, granularity: int = BOTH, launch_filter: int = ALL_LAUNCHES):
        self._ck(self.L.thermo_build_heatmap(self.h, granularity, launch_filter))

    def heatmap(self, object_id: int, granularity: int = WORD) -> np.ndarray:
        n = sz()
        self.L.thermo_query_heatmap(self.h, object_id, granularity, None, 0, ctypes.byref(n))
        out = np.zeros(n.value, dtype=np.uint32)
        self._ck(self.L.thermo_query_heatmap(self.h, object_id, granularity, out.ctypes.data, n.value,
                                             ctypes.byref(n)))
        return out

    def access(self, object_id: int) -> np.ndarray:
        """Lane accesses per word (thermo_query_access; track_access=True)."""
        n = sz()
        self.L.thermo_query_access(self.h, object_id, None, 0, ctypes.byref(n))
        out = np.zeros(n.value, dtype=np.uint32)
        self._ck(self.L.thermo_query_access(self.h, object_id, out.ctypes.data, n.value, ctypes.byref(n)))
        return out

    def runs(self, object_id: int):
        """Run-compressed rows (thermo_query_runs): (start [R], count [R], temps [R, 9])."""
        n = sz()
        self.L.thermo_query_runs(self.h, object_id, None, 0, ctypes.byref(n))
        raw = np.zeros((max(1, n.value), 14), dtype=np.uint32)  # 56-byte thermo_run
        self._ck(self.L.thermo_query_runs(self.h, object_id, raw.ctypes.data, n.value, ctypes.byref(n)))
        raw = raw[:n.value]
        start = raw[:, 0].astype(np.uint64) | (raw[:, 1].astype(np.uint64) << np.uint64(32))
        count = raw[:, 2].astype(np.uint64) | (raw[:, 3].astype(np.uint64) << np.uint64(32))
        return start, count, raw[:, 4:13].copy()

    def histogram(self, object_id: int, granularity: int) -> np.ndarray:
        out = np.zeros(LEVELS, dtype=np.uint64)
        self._ck(self.L.thermo_query_histogram(self.h, object_id, granularity, out.ctypes.data))
        return out

    def per_pc(self, granularity: int):
        n = sz()
        self.L.thermo_query_per_pc(self.h, granularity, None, 0, ctypes.byref(n))
        arr = (thermo_pc_hist * max(1, n.value))()
        self._ck(self.L.thermo_query_per_pc(self.h, granularity, arr, n.value, ctypes.byref(n)))
        return [(r.launch, r.pc, np.array(r.hist[:], dtype=np.uint64)) for r in arr[:n.value]]

    def classify(self, params: dict | None = None) -> list[dict]:
        p = thermo_params()
        self.L.thermo_default_params(ctypes.byref(p))
        for k, v in (params or {}).items():
            setattr(p, k, int(v))
        n = len(self.objects)
        arr = (thermo_indicators * n)()
        cnt = sz()
        self._ck(self.L.thermo_classify(self.h, ctypes.byref(p), arr, n, ctypes.byref(cnt)))
        out = []
        for r in arr[:cnt.value]:
            d = {f: int(getattr(r, f)) for f in IND_FIELDS}
            d["labels"] = int(r.labels)
            d["object_id"] = int(r.object_id)
            out.append(d)
        return out

    def stats(self) -> dict:
        s = thermo_stats()
        self._ck(self.L.thermo_get_stats(self.h, ctypes.byref(s)))
        d = {f: getattr(s, f) for f, _ in thermo_stats._fields_ if not f.startswith("reserved") and f != "ms_kernel"}
        d["ms_kernel"] = dict(zip(KERNELS, list(s.ms_kernel)))
        return d
