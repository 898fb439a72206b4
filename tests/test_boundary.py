"""The drop-in boundary (CPU, no GPU): the C-ABI library loads, exports every
entry point include/iqcc_b200.h declares, the Python binding covers all of
them, and errors are status codes (never a crash) when no device exists."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "iqcc_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(iqcc_gpu_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2603_08883_b200 import native
    lib = C.CDLL(native.LIB_PATH)
    missing = [s for s in declared() if not hasattr(lib, s)]
    assert not missing, f"not exported: {missing}"


def test_python_binding_covers_the_header():
    from paper_2603_08883_b200 import native
    assert set(declared()) == set(native.EXPORTED)


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2603_08883_b200", "libiqcc_b200.so")
    out = os.popen(f"cuobjdump --list-elf {so} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_errors_are_status_codes_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2603_08883_b200 import native
    rc = native.lib.iqcc_gpu_init(0)
    assert rc == native.IQCC_ECUDA
    assert b"CUDA" in native.lib.iqcc_gpu_last_error()
    h = C.c_void_p()
    rc = native.lib.iqcc_gpu_sum_create(4, None, None, 0, C.byref(h))
    assert rc == native.IQCC_ERUNTIME and b"iqcc_gpu_init" in native.lib.iqcc_gpu_last_error()


def test_shim_header_compiles_against_the_reference():
    """include/iqcc_b200/iqcc_gpu.hpp re-exposes namespace iqcc's hot-path
    API with the reference's own types; it must parse with them."""
    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc):
        pytest.skip("/root/reference absent")
    probe = os.path.join(ROOT, "tests", "cpp", "shim_compile_probe.cpp")
    rc = os.system(f"g++ -std=c++20 -fsyntax-only -I{ref_inc} -I{ROOT}/include {probe}")
    assert rc == 0
