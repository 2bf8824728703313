"""The reference's C++ API (include/multiproj/*.hpp) as a drop-in over the C-ABI.

CPU: the drop-in library builds, exports the reference symbols, and the
C++ test program (tests/cpp/dropin_test.cpp) compiles and links against it.
GPU: that program passes (reference worked examples + invariants).
"""
import os
import subprocess
import tempfile

import pytest

from paper_2405_02086_b200 import _build


@pytest.fixture(scope="module")
def cpp_test_binary():
    _build.build()
    out = os.path.join(tempfile.mkdtemp(), "dropin_test")
    return _build.build_cpp_test(out)


def test_dropin_exports_reference_api(cpp_test_binary):
    syms = subprocess.run(["nm", "-DC", "--defined-only", _build.DROPIN], capture_output=True, text=True).stdout
    for name in ["multiproj::bilevel_project(", "multiproj::bilevel_project_l1inf(", "multiproj::multilevel_project(",
                 "multiproj::multilevel_project_iter(", "multiproj::trilevel_project_l1infinf(",
                 "multiproj::multilevel_norm(", "multiproj::project_ball(", "multiproj::run_projection(",
                 "multiproj::parallel_project(", "multiproj::parse_norm_spec(", "multiproj::matrix_pq_norm(",
                 "multiproj::aggregate_leading_axis(", "multiproj::structured_sparsity(",
                 "multiproj::euclid_project_l1inf(", "multiproj::budget_oracle_grid(", "multiproj::clip_cost("]:
        assert name in syms, name
    assert os.access(cpp_test_binary, os.X_OK)


@pytest.mark.gpu
def test_dropin_cpp_suite_passes(cpp_test_binary):
    r = subprocess.run([cpp_test_binary], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK: 0 failure(s)" in r.stdout
