"""The reference's C++ API (include/multiproj/*.hpp) as a drop-in over the C-ABI.

CPU: the drop-in library builds, exports the reference symbols, and the
C++ test program (tests/cpp/dropin_test.cpp) compiles and links against it.
GPU: that program passes (reference worked examples + invariants).
"""
import os
import subprocess
import tempfile

import pytest

import numpy as np

from oracle import oracle as O
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
                 "multiproj::euclid_project_l1inf(", "multiproj::budget_oracle_grid(", "multiproj::clip_cost(",
                 "multiproj::read_tensor(", "multiproj::write_tensor(", "multiproj::tensor_checksum(",
                 "multiproj::bench_one(", "multiproj::run_radius_sweep(", "multiproj::project_file(",
                 "multiproj::read_csv_records(", "multiproj::write_csv_records(", "multiproj::measure_speedup("]:
        assert name in syms, name
    assert os.access(cpp_test_binary, os.X_OK)


@pytest.fixture(scope="module")
def io_binary():
    _build.build()
    return _build.build_io_test(os.path.join(tempfile.mkdtemp(), "io_compat"))


def _run(binary, *args):
    r = subprocess.run([binary, *map(str, args)], capture_output=True, text=True, timeout=120)
    return r.returncode, r.stdout.split()


needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_tensor_files_are_byte_compatible_with_the_reference(io_binary, tmp_path):
    """proj/src/tensor_io.cpp + rng.cpp: MLPT of orders 1-4 and CSV written by
    the reference read back by the drop-in (same checksum) and vice versa."""
    for k, shape in enumerate([(7,), (5, 3), (2, 3, 4), (2, 2, 3, 2), (13, 7)]):
        for ext in ([".mlpt", ".csv"] if len(shape) == 2 else [".mlpt"]):
            a, b = tmp_path / f"ref{k}{ext}", tmp_path / f"ours{k}{ext}"
            ck_ref = O.ref_write_uniform_tensor(a, shape, 100 + k)
            rc, out = _run(io_binary, "checksum", a)
            assert rc == 0 and int(out[0]) == ck_ref and int(out[1]) == int(np.prod(shape))
            rc, out = _run(io_binary, "write", b, 100 + k, -1.0, 1.0, *shape)
            assert rc == 0 and int(out[0]) == ck_ref
            assert O.ref_read_tensor_checksum(b) == (ck_ref, int(np.prod(shape)))
            if ext == ".mlpt":
                assert a.read_bytes() == b.read_bytes()


@needs_ref
def test_generator_and_records_match_the_reference(io_binary, tmp_path):
    rc, out = _run(io_binary, "rng", 7, 40)
    raw, nrm = O.ref_rng_stream(7, 40)
    assert rc == 0 and [int(v) for v in out[:40]] == [int(v) for v in raw]
    assert np.array_equal(np.array([float(v) for v in out[40:]]), nrm)
    src, dst = tmp_path / "rec.csv", tmp_path / "rec2.csv"
    O.ref_write_records_sample(src)
    rc, out = _run(io_binary, "records", src, dst)
    assert rc == 0 and out == ["2"]
    assert src.read_text() == dst.read_text()


def test_malformed_files_raise_ioerror(io_binary, tmp_path):  # proj/tests/test_io_rng.cpp:99-125
    (tmp_path / "bad.mlpt").write_bytes(b"NOPE")
    (tmp_path / "bad.csv").write_text("1.0,2.0\n3.0\n")
    (tmp_path / "nan.csv").write_text("1.0,abc\n")
    for f in ["missing.mlpt", "bad.mlpt", "bad.csv", "nan.csv"]:
        rc, out = _run(io_binary, "checksum", tmp_path / f)
        assert rc == 3 and out[0] == "IoError", (f, out)
    rc, out = _run(io_binary, "write", tmp_path / "t.mlpt", 1, -1.0, 1.0, 3, 3)
    data = (tmp_path / "t.mlpt").read_bytes()
    (tmp_path / "trunc.mlpt").write_bytes(data[:30])
    rc, out = _run(io_binary, "checksum", tmp_path / "trunc.mlpt")
    assert rc == 3 and out[0] == "IoError"
    rc, out = _run(io_binary, "write", tmp_path / "t3.csv", 1, -1.0, 1.0, 2, 2, 2)
    assert rc == 4 and out[0] == "ShapeError"


@pytest.mark.gpu
def test_dropin_cpp_suite_passes(cpp_test_binary):
    r = subprocess.run([cpp_test_binary], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK: 0 failure(s)" in r.stdout
