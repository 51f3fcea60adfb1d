"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper around the CPU oracle.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product package
(``paper_2507_18729_b200``) never imports it and shares no code with it.

The oracle itself (``thermo_oracle.cpp``) is a plain single-threaded C++17
implementation of the paper's definition (§IV-A1, §IV-B2):
an explicit ``std::set`` of warps per word.  See its header for citations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "thermo_oracle.cpp")
LIB = os.path.join(HERE, "liboracle.so")

ALL_LAUNCHES = 0xFFFFFFFF
LEVELS = 33

# indicator fields (order of the I_* enum in thermo_oracle.cpp)
IND_FIELDS = (
    "n_words", "n_sectors", "touched_sectors", "touched_words", "hot_sectors",
    "fs_sectors", "sum_x", "sum_x2_lo", "sum_x2_hi", "le1_words", "max_sector_count",
    "instrs", "misaligned_instrs", "gaps", "dom_gap", "dom_count", "labels",
)
# parameter order (P_* enum); defaults are SPEC's as exact rationals
PARAM_FIELDS = (
    "theta_hot", "alpha_num", "alpha_den", "beta_num", "beta_den", "fs_min",
    "smem_cap", "smem_cov_num", "smem_cov_den", "gamma_num", "gamma_den",
    "strided_min_sectors", "dom_num", "dom_den", "hot_frac_num", "hot_frac_den",
    "fs_frac_num", "fs_frac_den", "mis_frac_num", "mis_frac_den", "cv_num", "cv_den",
)
DEFAULT_PARAMS = dict(
    theta_hot=16, alpha_num=5, alpha_den=4, beta_num=4, beta_den=1, fs_min=4,
    smem_cap=1, smem_cov_num=9, smem_cov_den=10, gamma_num=1, gamma_den=2,
    strided_min_sectors=4, dom_num=3, dom_den=4, hot_frac_num=1, hot_frac_den=2,
    fs_frac_num=1, fs_frac_den=4, mis_frac_num=1, mis_frac_den=10, cv_num=1, cv_den=2,
)
LABELS = {
    "Hot": 1, "RandomHot": 2, "FalseSharing": 4, "SmemAbuseThreadLocal": 8,
    "SmemAbuseWarpPrivate": 16, "Misaligned": 32, "Strided": 64,
}


def label_names(bits: int) -> list[str]:
    return [k for k, v in LABELS.items() if bits & v]


class _Obj(ctypes.Structure):
    _fields_ = [("base", ctypes.c_uint64), ("len", ctypes.c_uint64),
                ("space", ctypes.c_uint32), ("id", ctypes.c_uint32)]


def build() -> str:
    """Compile the oracle (plain g++, no CUDA)."""
    if (not os.path.exists(LIB)) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", LIB, SRC])
    return LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        vp, sz, u32, u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint64
        L.orc_new.restype = vp
        L.orc_new.argtypes = [ctypes.POINTER(_Obj), sz]
        L.orc_free.argtypes = [vp]
        L.orc_restrict.argtypes = [vp, vp, vp, sz]
        L.orc_ingest.argtypes = [vp, vp, sz]
        L.orc_block_scope.argtypes = [vp, u32, u32]
        L.orc_launch_whitelist.argtypes = [vp, vp, ctypes.c_size_t]
        L.orc_ingest_warp.argtypes = [vp, vp, sz]
        L.orc_build.argtypes = [vp, u32]
        L.orc_word_counts.argtypes = [vp, u32, vp]
        L.orc_sector_counts.argtypes = [vp, u32, vp]
        L.orc_access_counts.argtypes = [vp, u32, vp]
        L.orc_runs.restype = sz
        L.orc_runs.argtypes = [vp, u32, vp, vp, vp, sz]
        L.orc_sample.argtypes = [vp, vp, vp, sz, vp]
        L.orc_hist.argtypes = [vp, u32, ctypes.c_int, vp]
        L.orc_n_pcs.restype = sz
        L.orc_n_pcs.argtypes = [vp]
        L.orc_pc_row.argtypes = [vp, sz, vp, vp, vp, vp]
        L.orc_stats.argtypes = [vp, vp]
        L.orc_classify.argtypes = [vp, vp, vp]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Oracle:
    """One oracle run: objects, then ingest calls, then build(launch_filter).

    objects: list of (base, len, space, id) in registration order; results are
    indexed by that order (object index), not by id.
    """

    def __init__(self, objects):
        L = _load()
        self.objects = [tuple(int(x) for x in o[:4]) for o in objects]
        arr = (_Obj * len(self.objects))(*[_Obj(*o) for o in self.objects])
        self._h = L.orc_new(arr, len(self.objects))

    def close(self):
        h = getattr(self, "_h", None)
        self._h = None
        if h and _lib is not None:
            try:
                _lib.orc_free(h)
            except Exception:  # interpreter shutdown
                pass

    __del__ = close

    def restrict(self, obj_idx, sectors):
        oi = np.ascontiguousarray(obj_idx, dtype=np.uint32)
        se = np.ascontiguousarray(sectors, dtype=np.uint64)
        _load().orc_restrict(self._h, _ptr(oi), _ptr(se), len(oi))

    def ingest_warp(self, records):
        """Warp-instruction records (272 bytes each; int32 [n, 68]) as one call."""
        a = np.ascontiguousarray(_as_numpy(records))
        assert a.nbytes % 272 == 0
        _load().orc_ingest_warp(self._h, _ptr(a), a.nbytes // 272)

    def block_scope(self, warps_per_block: int, block: int):
        """Keep only the records of one sampled block; call before ingest."""
        _load().orc_block_scope(self._h, warps_per_block, block)

    def launch_whitelist(self, launches):
        """Kernel sampling by whitelist: only these launches are traced
        (empty: all); call before ingest."""
        a = np.ascontiguousarray(np.asarray(list(launches), dtype=np.uint32))
        _load().orc_launch_whitelist(self._h, _ptr(a) if len(a) else None, len(a))

    def ingest(self, records):
        """records: anything exposing 16-byte records (numpy/torch int32 [n,4])."""
        a = np.ascontiguousarray(_as_numpy(records))
        assert a.nbytes % 16 == 0
        _load().orc_ingest(self._h, _ptr(a), a.nbytes // 16)

    def build(self, launch_filter: int = ALL_LAUNCHES):
        _load().orc_build(self._h, launch_filter)

    def n_words(self, o):
        return (self.objects[o][1] + 3) // 4

    def n_sectors(self, o):
        return (self.objects[o][1] + 31) // 32

    def word_counts(self, o) -> np.ndarray:
        out = np.zeros(self.n_words(o), dtype=np.uint32)
        _load().orc_word_counts(self._h, o, _ptr(out))
        return out

    def sector_counts(self, o) -> np.ndarray:
        out = np.zeros(self.n_sectors(o), dtype=np.uint32)
        _load().orc_sector_counts(self._h, o, _ptr(out))
        return out

    def access_counts(self, o) -> np.ndarray:
        """Lane accesses per word of object index o, all launches (G27)."""
        out = np.zeros(self.n_words(o), dtype=np.uint32)
        _load().orc_access_counts(self._h, o, _ptr(out))
        return out

    def runs(self, o):
        """Run-compressed rows of object index o: (start [R], count [R], temps [R, 9])."""
        L = _load()
        n = L.orc_runs(self._h, o, None, None, None, 0)
        st = np.zeros(n, dtype=np.uint64)
        ct = np.zeros(n, dtype=np.uint64)
        tp = np.zeros((n, 9), dtype=np.uint32)
        L.orc_runs(self._h, o, _ptr(st), _ptr(ct), _ptr(tp), n)
        return st, ct, tp

    def sample(self, obj_idx, sectors) -> np.ndarray:
        oi = np.ascontiguousarray(obj_idx, dtype=np.uint32)
        se = np.ascontiguousarray(sectors, dtype=np.uint64)
        out = np.zeros((len(oi), 9), dtype=np.uint32)
        _load().orc_sample(self._h, _ptr(oi), _ptr(se), len(oi), _ptr(out))
        return out

    def hist(self, o, sector: bool) -> np.ndarray:
        out = np.zeros(LEVELS, dtype=np.uint64)
        _load().orc_hist(self._h, o, int(bool(sector)), _ptr(out))
        return out

    def per_pc(self):
        L = _load()
        rows = []
        for i in range(L.orc_n_pcs(self._h)):
            la, pc = ctypes.c_uint32(), ctypes.c_uint32()
            hw = np.zeros(LEVELS, dtype=np.uint64)
            hs = np.zeros(LEVELS, dtype=np.uint64)
            L.orc_pc_row(self._h, i, ctypes.byref(la), ctypes.byref(pc), _ptr(hw), _ptr(hs))
            rows.append((la.value, pc.value, hw, hs))
        return rows

    def stats(self) -> dict:
        out = np.zeros(4, dtype=np.uint64)
        _load().orc_stats(self._h, _ptr(out))
        return dict(records=int(out[0]), invalid=int(out[1]),
                    unmapped_words=int(out[2]), mapped_word_accesses=int(out[3]))

    def classify(self, params: dict | None = None) -> list[dict]:
        p = dict(DEFAULT_PARAMS)
        p.update(params or {})
        prm = np.array([p[k] for k in PARAM_FIELDS], dtype=np.uint64)
        out = np.zeros((len(self.objects), len(IND_FIELDS)), dtype=np.uint64)
        _load().orc_classify(self._h, _ptr(prm), _ptr(out))
        return [{k: int(v) for k, v in zip(IND_FIELDS, row)} for row in out]


def _as_numpy(records) -> np.ndarray:
    try:
        import torch
        if isinstance(records, torch.Tensor):
            return records.detach().cpu().contiguous().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(records)


def run(objects, chunks, launch_filter=ALL_LAUNCHES) -> Oracle:
    """Convenience: build an oracle over `chunks` (list of record arrays)."""
    o = Oracle(objects)
    for c in chunks:
        o.ingest(c)
    o.build(launch_filter)
    return o
