"""CPU checks of the boundary: libsbmds.so builds for sm_100a, loads, exports every symbol
include/sbmds.h declares, and carries tcgen05/TMA-era SASS for sm_100a. No compute calls."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sbmds.h")


@pytest.fixture(scope="module")
def libpath():
    from paper_1705_10887_b200 import build
    return build.build()


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sbmds_[a-z_]+)\s*\(", src)))


def test_header_functions_match_binding():
    from paper_1705_10887_b200._lib import EXPORTS
    assert header_functions() == sorted(EXPORTS)


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for fn in header_functions():
        assert fn in syms, fn


def test_library_loads_and_answers_without_gpu(libpath):
    from paper_1705_10887_b200._lib import lib
    L = lib()
    assert L.sbmds_abi_version() == 2
    assert L.sbmds_launch_count() >= 0
    assert isinstance(L.sbmds_last_error(), bytes)


def test_invalid_arguments_rejected_before_any_device_work(libpath):
    import ctypes
    from paper_1705_10887_b200._lib import lib, SBMDS_EINVAL
    L = lib()
    h = ctypes.c_void_p()
    assert L.sbmds_create(0, 0, 0, None, None, None, None, 0, None, ctypes.byref(h)) == SBMDS_EINVAL
    assert L.sbmds_create(10, 11, 0, None, None, None, None, 0, None, ctypes.byref(h)) == SBMDS_EINVAL
    assert b"l <= n" in L.sbmds_last_error()
    assert L.sbmds_apply(None, 4, None, None, None) == SBMDS_EINVAL
    L.sbmds_destroy(None)   # NULL-safe


def test_sass_is_sm100a_with_tma(libpath):
    out = subprocess.run(["cuobjdump", "-lelf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    fn = [blk for blk in sass.split("Function : ") if blk.startswith("_ZN5sbmds14k_dstream_ffma")]
    assert fn and all("UTMALDG" in blk and "UBLKCP" in blk for blk in fn)


def test_product_has_no_oracle_or_fallback_imports():
    """The product package never imports the oracle, and has no CPU/torch math fallback."""
    pkg = os.path.join(ROOT, "paper_1705_10887_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in src.replace("oracle.", "").split("import")[0] or "import oracle" not in src
            assert "from oracle" not in src and "import oracle" not in src
            assert "scipy" not in src


def test_sbha_p_matches_the_oracle_rule(libpath):
    """sbmds_sbha_p (host arithmetic, no GPU): p = clamp(ceil((n - l) p_row / l), 1, n - l), the rule
    the sBHA oracle states (ceiling per SPEC.md:380), on a grid including the SPEC
    example n = 100, l = 20, p_row = 10 -> 40, fractional p_row and the clamps."""
    from oracle import sbha_oracle as B
    from paper_1705_10887_b200._lib import lib
    L = lib()
    assert L.sbmds_sbha_p(100, 20, 10.0) == 40
    for n in (2, 10, 101, 2000, 100_000, 1_800_000):
        for l in sorted({1, 2, n // 7 or 1, n // 2 or 1, n - 1}):
            if not 1 <= l < n:
                continue
            for prow in (0.5, 1.0, 3.0, 8.0, 16.0, 33.3, 1e9):
                assert L.sbmds_sbha_p(n, l, prow) == B.p_from_prow(n, l, prow), (n, l, prow)
    assert L.sbmds_sbha_p(10, 10, 4.0) < 0 and L.sbmds_sbha_p(10, 3, 0.0) < 0
