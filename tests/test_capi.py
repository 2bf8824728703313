"""CPU-side checks of the drop-in boundary (no GPU compute):

* libmp_b200.so loads and exports every function include/mp_cuda.h declares;
* argument validation mirrors the reference exception taxonomy
  (proj/include/multiproj/errors.hpp; proj/src/bilevel.cpp:12-14,
  proj/src/multilevel.cpp:45-53) and happens before any device work;
* workspace sizing is well defined;
* datagen restates the reference generator bit-exactly.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2405_02086_b200 as mp
from paper_2405_02086_b200 import _capi, datagen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "mp_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mp_[a-z_]+)\s*\(", src)))


def test_header_and_exports_agree():
    declared = header_functions()
    assert sorted(_capi.EXPORTS) == declared
    L = _capi.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert L.mp_version() >= 100


def test_status_codes_mirror_reference():
    L = _capi.lib()
    buf = (C.c_char * 64)()
    # eta < 0 -> ValueError (proj/src/bilevel.cpp:13-14)
    st = L.mp_bilevel_project(buf, buf, 0, 2, 2, 0, 2, -1.0, None, None, None, 0, buf, 64, None)
    assert st == _capi.MP_ERR_VALUE
    st = L.mp_bilevel_project(buf, buf, 0, 2, 2, 0, 2, float("nan"), None, None, None, 0, buf, 64, None)
    assert st == _capi.MP_ERR_VALUE
    # empty matrix -> ShapeError (proj/src/tensor.cpp:23-31)
    assert L.mp_bilevel_project(buf, buf, 0, 0, 2, 0, 2, 1.0, None, None, None, 0, buf, 64, None) == _capi.MP_ERR_SHAPE
    # bad norm / dtype codes -> ConfigError
    assert L.mp_bilevel_project(buf, buf, 0, 2, 2, 7, 2, 1.0, None, None, None, 0, buf, 64, None) == _capi.MP_ERR_CONFIG
    assert L.mp_bilevel_project(buf, buf, 9, 2, 2, 0, 2, 1.0, None, None, None, 0, buf, 64, None) == _capi.MP_ERR_CONFIG
    # too-small workspace is reported, not overrun
    assert L.mp_bilevel_project(buf, buf, 0, 2, 2, 0, 2, 1.0, None, None, None, 0, buf, 64, None) == _capi.MP_ERR_WORKSPACE
    assert b"workspace" in L.mp_last_error()


def test_multilevel_validation_order():
    L = _capi.lib()
    buf = (C.c_char * 64)()
    shape = (C.c_int64 * 2)(2, 2)
    lv1 = (C.c_int * 1)(0)
    lv3 = (C.c_int * 3)(2, 2, 0)
    # depth 0 -> ConfigError; depth != order -> ShapeError (proj/src/multilevel.cpp:45-53)
    assert L.mp_multilevel_project(buf, buf, 0, shape, 2, lv1, 0, 1.0, None, None, 0, buf, 64, None) == _capi.MP_ERR_CONFIG
    assert L.mp_multilevel_project(buf, buf, 0, shape, 2, lv1, 1, 1.0, None, None, 0, buf, 64, None) == _capi.MP_ERR_SHAPE
    assert L.mp_multilevel_project(buf, buf, 0, shape, 2, lv3, 3, 1.0, None, None, 0, buf, 64, None) == _capi.MP_ERR_SHAPE
    zero = (C.c_int64 * 2)(2, 0)
    assert L.mp_multilevel_project(buf, buf, 0, zero, 2, lv3, 2, 1.0, None, None, 0, buf, 64, None) == _capi.MP_ERR_SHAPE


def test_python_mirror_errors_without_gpu():
    with pytest.raises(ValueError):
        mp.parse_norm_spec("inf,bogus")  # proj/tests/python/test_smoke.py:71-75
    with pytest.raises(ValueError):
        mp.parse_norm_spec("")  # proj/tests/test_multilevel.cpp:17
    assert mp.parse_norm_spec("inf,inf,1") == [2, 2, 0]
    with pytest.raises(mp.MpShapeError):
        mp.bilevel_project(np.ones(3), 1.0)
    with pytest.raises(mp.MpShapeError):
        mp.trilevel_project_l1infinf(np.ones((2, 2)), 1.0)


def test_workspace_sizes():
    L = _capi.lib()
    for dt in (0, 1):
        for q in (0, 1, 2):
            w = L.mp_bilevel_workspace_size(dt, 10000, 10000, 0, q)
            assert 0 < w < 64 << 20
    assert L.mp_bilevel_workspace_size(0, 0, 5, 0, 2) == 0
    shape = (C.c_int64 * 3)(256, 256, 256)
    lv = (C.c_int * 3)(2, 2, 0)
    assert L.mp_multilevel_workspace_size(0, shape, 3, lv, 3) > 0
    assert L.mp_project_ball_workspace_size(0, 10 ** 6, 0) > 10 ** 6 * 8


def test_datagen_restates_reference_rng(golden):
    assert np.array_equal(datagen.raw(7, 64), golden["rng_raw_seed7"])
    assert np.array_equal(datagen.uniform(2, 64, -1.0, 1.0, dtype=np.float64), golden["rng_uniform_seed2"])
    assert np.array_equal(datagen.normal(1, 64, dtype=np.float64), golden["rng_normal_seed1"])
    u32 = datagen.uniform(2, (8, 8), -1.0, 1.0)
    assert u32.dtype == np.float32
    assert np.array_equal(u32.reshape(-1), golden["rng_uniform_seed2"].astype(np.float32))


def test_config5_eta_zeroes_target_fraction():
    v = np.abs(datagen.laplace(5, (64, 512), 0.01)).max(axis=0).astype(np.float64)
    eta = datagen.config5_eta(v)
    from oracle import oracle as O
    u = O.project_ball(v, "1", eta)
    assert int(np.sum(u == 0)) == int(np.floor(0.9 * 512)) + 1


def test_device_projectors_reject_unsupported_dtypes():
    """float16 / bfloat16 / integer tensors must never reach the kernels (they
    would read and write 8-byte elements through a smaller buffer)."""
    import torch
    for dt in (torch.float16, torch.bfloat16, torch.int32, torch.int64, "float16"):
        with pytest.raises(mp.MpConfigError):
            mp.BilevelProjector(8, 8, dt)
        with pytest.raises(mp.MpConfigError):
            mp.MultilevelProjector((4, 4, 4), "inf,inf,1", dt)
    with pytest.raises(mp.MpConfigError):
        mp.BilevelProjector(8, 8, torch.float32, device="cpu")
