"""Host-side checks of the C ABI that need no GPU: the library loads, exports
every entry point include/tca.h declares, and validates arguments before
touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "tca.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(tca_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    from paper_1001_5460_b200 import tca
    syms = _header_symbols()
    assert len(syms) >= 12
    lib = ctypes.CDLL(tca.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(tca.EXPORTED)
    assert "sm_100a" in tca.version()


def test_status_strings():
    from paper_1001_5460_b200 import tca
    for code in range(10):
        assert tca._lib.tca_status_string(code).decode().startswith("TCA_")


@pytest.mark.parametrize("case", ["order0", "order5", "neg_lambda", "nan_lambda", "zero_extent",
                                  "nan_A", "bad_dtype"])
def test_create_validates_before_any_launch(case):
    from paper_1001_5460_b200 import tca
    A = [np.eye(3)] * 3
    kw = dict(A=A, L=None, lam=0.1, dtype="f64")
    order_override = None
    if case == "order0":
        order_override = 0
    elif case == "order5":
        order_override = 5
    elif case == "neg_lambda":
        kw["lam"] = -1.0
    elif case == "nan_lambda":
        kw["lam"] = float("nan")
    elif case == "zero_extent":
        kw["A"] = [np.zeros((3, 0))] * 3
    elif case == "nan_A":
        kw["A"] = [np.full((3, 3), np.nan)] * 3
    if order_override is not None or case == "bad_dtype":
        h = ctypes.c_void_p()
        n = (ctypes.c_int64 * 4)(3, 3, 3, 3)
        dp = ctypes.POINTER(ctypes.c_double)
        arrs = [np.eye(3) for _ in range(4)]
        Ap = (dp * 4)(*[a.ctypes.data_as(dp) for a in arrs])
        st = tca._lib.tca_operator_create(ctypes.byref(h), 3 if order_override is None else order_override,
                                          n, n, Ap, None, 0.1, 7 if case == "bad_dtype" else 0, None, None)
        assert st == tca.ERR_INVALID_ARG
        assert not h.value
        assert tca._lib.tca_last_error().decode()
        return
    with pytest.raises(tca.TcaError) as ei:
        tca.Operator(**kw)
    assert ei.value.status in (tca.ERR_INVALID_ARG, tca.ERR_SHAPE)


def test_null_operator_calls_fail_cleanly():
    from paper_1001_5460_b200 import tca
    assert tca._lib.tca_apply(None, None, None, None) == tca.ERR_INVALID_ARG
    assert tca._lib.tca_rhs(None, None, None, None) == tca.ERR_INVALID_ARG
    for x0_zero in (0, 1):
        for fn in (tca._lib.tca_cg_solve, tca._lib.tca_pcg_solve, tca._lib.tca_cgsr_solve):
            assert fn(None, None, None, x0_zero, 0.0, 1, None, None) == tca.ERR_INVALID_ARG
    assert tca._lib.tca_generate_normal(None, 0, 5, 0, 1, 0, 1.0, None) == tca.ERR_INVALID_ARG
    assert tca._lib.tca_jacobi_solve(None, None, None, 0.0, 1, None, None) == tca.ERR_INVALID_ARG
    assert tca._lib.tca_precond_apply(None, None, None, None) == tca.ERR_INVALID_ARG
    assert tca._lib.tca_operator_create_gram(None, 3, None, None, None, 1.0, 0, None, None) == tca.ERR_INVALID_ARG
    assert tca._lib.tca_solve_host_batch(None, 1, None, None, 0.0, 1, None, None) == tca.ERR_INVALID_ARG
    assert tca._lib.tca_operator_cg_fused_step(None) == -1
    assert tca._lib.tca_operator_cg_deferred_x(None) == -1
    assert tca._lib.tca_operator_cg_engine(None) == -1
    tca._lib.tca_operator_destroy(None)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1001_5460_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src), f


@pytest.mark.parametrize("case", ["t_above", "t_below", "t_nan", "neg_K", "null_t", "L_nan", "order0"])
def test_create_scattered_validates_before_any_launch(case):
    """tca_operator_create_scattered rejects bad input before touching the device
    (so it runs without a GPU): sample coordinates outside [0, n_d - 1] or not
    finite, K < 0, t NULL with K > 0, non-finite L, bad order."""
    from paper_1001_5460_b200 import tca
    dp = ctypes.POINTER(ctypes.c_double)
    n = (6, 5, 4)
    t = np.array([[1.0, 2.0, 3.0], [0.5, 0.5, 0.5]])
    K, order = t.shape[0], 3
    L = [np.eye(k - 2, k) for k in n]
    if case == "t_above":
        t[1, 2] = 3.5
    elif case == "t_below":
        t[0, 0] = -1e-9
    elif case == "t_nan":
        t[1, 1] = np.nan
    elif case == "neg_K":
        K = -1
    elif case == "L_nan":
        L[1] = L[1].copy()
        L[1][0, 0] = np.inf
    elif case == "order0":
        order = 0
    h = ctypes.c_void_p()
    n_arr = (ctypes.c_int64 * 3)(*n)
    L_arr = (dp * 3)(*[np.ascontiguousarray(l).ctypes.data_as(dp) for l in L])
    tp = None if case == "null_t" else np.ascontiguousarray(t).ctypes.data_as(dp)
    st = tca._lib.tca_operator_create_scattered(ctypes.byref(h), order, n_arr, K, tp, L_arr, 0.1, 0, None)
    assert st == tca.ERR_INVALID_ARG
    assert not h.value
    assert tca._lib.tca_last_error().decode()
