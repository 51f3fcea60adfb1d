"""paper_2507_18729_b200 -- libthermo, a B200-native heat-map reduction.

The data-parallel hot path of cuThermo (arXiv 2507.18729): a GPU memory-access
trace -> per-word and per-sector distinct-warp counts for every registered
object -> heat-level histograms per object and per PC -> pattern indicators.
The compute lives in ``libthermo.so`` (sm_100a CUDA, C ABI in include/thermo.h);
``thermo`` is its ctypes binding.
"""
from .thermo import (ALL_LAUNCHES, BOTH, DEDUP_AUTO, DEDUP_DENSE, DEDUP_HASH, DEDUP_SEGMENT, DEDUP_SORT,  # noqa: F401
                     LABELS, LEVELS, SECTOR, WORD,
                     Thermo, ThermoError, default_params, label_names, load)

__all__ = ["Thermo", "ThermoError", "load", "default_params", "label_names", "WORD", "SECTOR", "BOTH",
           "ALL_LAUNCHES", "DEDUP_AUTO", "DEDUP_SORT", "DEDUP_HASH", "DEDUP_SEGMENT", "DEDUP_DENSE", "LEVELS",
           "LABELS"]
