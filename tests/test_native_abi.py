"""The C ABI library: loads without a GPU, exports every symbol the header
declares, and the ctypes signature table covers them all.  CPU only."""

import os
import re
import subprocess

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pif_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(pif_\w+)\s*\(", text,
                                 re.M)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("pif_plan_create", "pif_bin_keys", "pif_bin_scatter", "pif_spread_sorted",
              "pif_grid_to_modes", "pif_solve_fields", "pif_interp_push", "pif_interp_sorted"):
        assert s in syms


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2605_10729_b200 import _native
    lib = _native.load()
    assert lib.pif_abi_version() == 1
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (pif_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_ctypes_table_matches_header():
    from paper_2605_10729_b200 import _native
    assert sorted(_native.SIGNATURES) == declared_symbols()


def test_library_is_sm100a():
    from paper_2605_10729_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_hot_kernels_use_fp64_tensor_cores():
    """The fused spread / gather kernels are DMMA (fp64 mma.sync) kernels."""
    from paper_2605_10729_b200 import _native
    out = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "DMMA.8x8x4" in out
    assert "REDG.E.ADD.F64" in out


def test_errors_map_to_python_exceptions():
    import ctypes

    import pytest

    from paper_2605_10729_b200 import _native
    lib = _native.load()
    h = ctypes.c_void_p()
    with pytest.raises(ValueError):
        _native.check(lib.pif_plan_create(None, 0, ctypes.byref(h)), "pif_plan_create")


def test_interior_weight_polynomials_are_accurate():
    """Host-side check of the polynomial window weights every plan builds."""
    import ctypes

    from paper_2605_10729_b200 import _native
    lib = _native.load()
    for w in range(2, 15):            # DMMA kernels (w <= 8) and ring kernels (9..14)
        err = (ctypes.c_double * 3)()
        mask = ctypes.c_int()
        _native.check(lib.pif_es_poly_info(w, 2.30 * w, err, ctypes.byref(mask)))
        if w >= 6:                     # eps <= 1e-5: every interior weight is a polynomial
            assert mask.value == 0, (w, mask.value)
        assert err[0] <= 4e-15, (w, err[0])   # polynomials in use meet the bound


def test_no_unresolved_symbols_of_our_own():
    from paper_2605_10729_b200 import _native
    out = subprocess.run(["nm", "-D", "--undefined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "pif" not in out, out


def test_product_path_fails_loudly_without_the_extension_or_a_gpu():
    """No CPU fallback: a missing libpifb200.so raises on load, and the operator
    API refuses to run without a CUDA device (this container has none)."""
    import subprocess
    import sys
    code = ("import paper_2605_10729_b200._native as n\n"
            "try:\n    n.load()\nexcept ImportError as e:\n    print('raised', 'no CPU fallback' in str(e))\n")
    env = dict(os.environ, PIF_B200_LIB="/nonexistent/libpifb200.so")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=ROOT).stdout
    assert "raised True" in out, out
    import numpy as np
    import pytest
    import torch

    import paper_2605_10729_b200 as pb
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    plan = pb.make_plan(8, 1.0, 1e-7)
    with pytest.raises(RuntimeError, match="no CPU implementation"):
        pb.type1(plan, np.zeros((4, 3)), np.ones(4))
