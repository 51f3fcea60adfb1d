"""Build libthermo.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2507_18729_b200.build          # incremental
    python -m paper_2507_18729_b200.build --force

Objects go to paper_2507_18729_b200/build/, the shared library to
paper_2507_18729_b200/libthermo.so (git-ignored, shipped with gpurun).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJDIR = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libthermo.so")
SOURCES = ["decode.cu", "decode_fast.cu", "decode_lane.cu", "decode_warp.cu", "sort.cu", "segment.cu", "dense.cu", "count.cu", "indicators.cu", "shard.cu", "export.cu", "thermo_api.cu"]
HEADERS = ["thermo_internal.cuh", "decode_common.cuh", "shard.cuh", os.path.join("..", "..", "include", "thermo.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-Xptxas", "-v,-warn-spills", f"-I{os.path.join(ROOT, 'include')}"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    hdr_t = max(_mtime(os.path.join(CSRC, h)) for h in HEADERS)
    objs, todo = [], []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        op = os.path.join(OBJDIR, src.replace(".cu", ".o"))
        objs.append(op)
        if force or _mtime(op) < max(_mtime(sp), hdr_t):
            todo.append((src, [NVCC, *ARCH, *FLAGS, "-c", sp, "-o", op]))

    def compile_one(item):
        return item[0], subprocess.run(item[1], capture_output=True, text=True)

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, todo))
    for src, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
    rebuilt = bool(todo)
    if force or rebuilt or not os.path.exists(LIB):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcuda", "-lnccl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
