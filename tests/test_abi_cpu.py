"""CPU-side checks of the boundary: the library builds for sm_100a, loads, and
exports every symbol include/thermo.h declares (no compute calls without a GPU).
Also the host-only pieces: defaults, struct layouts and the product's
independence from the oracle."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "thermo.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(thermo_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2507_18729_b200 import build as B
    B.build()
    from paper_2507_18729_b200 import thermo
    return thermo.load()


def test_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    from paper_2507_18729_b200 import thermo
    assert set(thermo.EXPORTS) == set(syms)


def test_sm100a_cubin_present():
    import subprocess
    from paper_2507_18729_b200 import build as B
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_defaults(lib):
    from paper_2507_18729_b200 import thermo
    cfg = thermo.thermo_config()
    lib.thermo_default_config(ctypes.byref(cfg))
    assert (cfg.max_launches, cfg.max_pcs, cfg.track_pc) == (1, 4096, 1)
    p = thermo.default_params()
    import oracle
    assert p == oracle.DEFAULT_PARAMS   # same S:347 defaults on both sides
    assert lib.thermo_abi_version() == 6


def test_struct_sizes():
    from paper_2507_18729_b200 import thermo
    assert ctypes.sizeof(thermo.thermo_object) == 24
    assert ctypes.sizeof(thermo.thermo_config) == 40
    assert ctypes.sizeof(thermo.thermo_params) == 22 * 8
    assert ctypes.sizeof(thermo.thermo_indicators) == 8 + 16 * 8
    assert ctypes.sizeof(thermo.thermo_pc_hist) == 8 + 33 * 8
    assert ctypes.sizeof(thermo.thermo_stats) == 10 * 8 + 8 + 9 * 8 + 8 + 16 + 9 * 8 + 16  # + ms_kernel[9], local_sectors, local_keys (ABI 5)


def test_create_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2507_18729_b200 import thermo
    with pytest.raises(thermo.ThermoError):
        thermo.Thermo()


def test_product_does_not_touch_oracle():
    """The product package never imports, links or reads oracle/ or /root/reference."""
    pkg = os.path.join(ROOT, "paper_2507_18729_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "/root/reference" not in txt, f


def test_dense_dedup_needs_sampled_block_mode(lib):
    """THERMO_DEDUP_DENSE is rejected before any device call
    unless 1 <= block_warps <= 64 (the paper's warp bitmask holds <= 64 warps)."""
    from paper_2507_18729_b200 import thermo
    EINVAL = -1
    for bw in (0, 65, 1024):
        cfg = thermo.thermo_config()
        lib.thermo_default_config(ctypes.byref(cfg))
        cfg.dedup, cfg.block_warps = thermo.DEDUP_DENSE, bw
        h = ctypes.c_void_p()
        assert lib.thermo_create(ctypes.byref(h), 0, None, ctypes.byref(cfg)) == EINVAL
    cfg = thermo.thermo_config()
    lib.thermo_default_config(ctypes.byref(cfg))
    cfg.dedup = 5  # past the last mode
    assert lib.thermo_create(ctypes.byref(ctypes.c_void_p()), 0, None, ctypes.byref(cfg)) == EINVAL
