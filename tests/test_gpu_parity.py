"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Small and medium sizes are compared element-wise with the §8(c) rule
(tests/parity.py); BASELINE.json full sizes are checked element-wise where the
oracle finishes in seconds and otherwise through size-independent properties
(feasibility, idempotence, determinism, in-place == out-of-place).
"""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2405_02086_b200 as mp
from oracle import oracle as O
from paper_2405_02086_b200 import datagen
from tests.parity import check_bilevel, check_multilevel

pytestmark = pytest.mark.gpu

bit_equal = lambda a, b: np.array_equal(np.ascontiguousarray(a).view(np.uint8), np.ascontiguousarray(b).view(np.uint8))
NORMS = ["1", "2", "inf"]


def oracle_bilevel(y32, eta, p="1", q="inf"):
    return O.bilevel(np.asarray(y32, np.float64), eta, p, q)


def run(y, eta, p="1", q="inf", flags=0):
    x, budgets, z = mp.bilevel_project(y, eta, p, q, flags=flags)
    return x, np.asarray(budgets), z


# ---------------------------------------------------------------- goldens
def test_golden_bilevel_f64(golden):
    """f64 device path vs the compiled reference's own outputs."""
    for i in range(int(golden["bi_count"][0])):
        y = golden[f"bi{i}_y"].astype(np.float64)
        p, q, eta = golden[f"bi{i}_meta"]
        p, q = int(p), int(q)
        x, b, z = run(y, eta, p, q)
        xr, br = golden[f"bi{i}_x"], golden[f"bi{i}_b"]
        np.testing.assert_allclose(b, br, rtol=1e-12, atol=1e-300, err_msg=f"case {i}")
        np.testing.assert_allclose(x, xr, rtol=1e-12, atol=1e-15, err_msg=f"case {i}")
        assert z == golden[f"bi{i}_z"][0], i


def test_golden_bilevel_f32(golden):
    """fp32 device path vs the reference (f64 on the same fp32 values)."""
    for i in range(int(golden["bi_count"][0])):
        y32 = golden[f"bi{i}_y"]
        p, q, eta = golden[f"bi{i}_meta"]
        qs = NORMS[int(q)]
        x, b, z = run(y32, eta, int(p), int(q))
        assert x.dtype == np.float32
        ref = oracle_bilevel(y32, eta, NORMS[int(p)], qs)
        assert bit_equal(ref["X"], golden[f"bi{i}_x"])
        check_bilevel(x, y32, ref, qs, zero_cols_gpu=z)


def test_golden_multilevel(golden):
    for i in range(int(golden["ml_count"][0])):
        t = golden[f"ml{i}_t"]
        lv = [int(k) for k in golden[f"ml{i}_lv"]]
        eta = float(golden[f"ml{i}_eta"][0])
        x64, chain = mp.multilevel_project(t.astype(np.float64), lv, eta, return_chain=True)
        np.testing.assert_allclose(x64, golden[f"ml{i}_x"], rtol=1e-12, atol=1e-15, err_msg=f"case {i}")
        flat = np.concatenate([c.reshape(-1) for c in chain]) if chain else np.zeros(0)
        np.testing.assert_allclose(flat, golden[f"ml{i}_chain"], rtol=1e-12, atol=1e-15, err_msg=f"case {i}")
        x32, chain32 = mp.multilevel_project(t, lv, eta, return_chain=True)
        assert x32.dtype == np.float32
        if len(lv) >= 2:  # the per-level §8(c) rule, no absolute slack
            ref_chain = _split_chain(golden[f"ml{i}_chain"], t.shape)
            check_multilevel(x32, t, lv, golden[f"ml{i}_x"], ref_chain, chain32)
        else:
            np.testing.assert_allclose(x32, golden[f"ml{i}_x"], rtol=1e-5, atol=0.0, err_msg=f"case {i}")


def _split_chain(flat, shape):
    out, off = [], 0
    for i in range(len(shape) - 1, 0, -1):
        size = int(np.prod(shape[i:]))
        out.append(np.asarray(flat[off:off + size]).reshape(shape[i:]))
        off += size
    return out


MULTI_SPECS_3D = ["1,1,1", "2,inf,1", "inf,1,1", "1,inf,1", "2,2,1", "inf,2,1", "1,1,2"]


@pytest.mark.parametrize("spec", MULTI_SPECS_3D)
@pytest.mark.parametrize("d", [128, 256])
def test_multilevel_f32_nontrivial_specs(spec, d):
    """fp32 non-collapsed multi-level specs at size, per-level §8(c) rule
    against the oracle on the same fp32 values (upcast to f64)."""
    t = datagen.normal(400 + d, (d, d, d))
    t64 = t.astype(np.float64)
    levels = spec.split(",")
    codes = [mp.norm_code(q) for q in levels]
    eta = 0.05 * O.multilevel_norm(t64, levels)
    x, chain = mp.multilevel_project(t, spec, eta, return_chain=True)
    xr, chain_r = O.multilevel(t64, levels, eta, want_chain=True)
    rep = check_multilevel(x, t, codes, xr, chain_r, chain)
    assert rep["max_rel"] < 1e-5


@pytest.mark.parametrize("shape", [(16, 24, 32, 48), (32, 32, 32, 32)])
@pytest.mark.parametrize("spec", ["1,2,inf,1", "inf,1,2,1", "2,1,1,1"])
def test_multilevel_f32_order4(shape, spec):
    t = datagen.normal(77, shape)
    t64 = t.astype(np.float64)
    levels = spec.split(",")
    codes = [mp.norm_code(q) for q in levels]
    eta = 0.05 * O.multilevel_norm(t64, levels)
    x, chain = mp.multilevel_project(t, spec, eta, return_chain=True)
    xr, chain_r = O.multilevel(t64, levels, eta, want_chain=True)
    check_multilevel(x, t, codes, xr, chain_r, chain)


def test_golden_vector_balls(golden):
    for i in range(int(golden["vb_count"][0])):
        y = golden[f"vb{i}_y"].astype(np.float64)
        q, r = golden[f"vb{i}_meta"]
        x = mp.project_ball(y, int(q), r)
        np.testing.assert_allclose(x, golden[f"vb{i}_x"], rtol=1e-12, atol=1e-15, err_msg=f"case {i}")


# --------------------------------------------------- known answers (API)
def test_reference_smoke_examples():  # proj/tests/python/test_smoke.py
    np.testing.assert_allclose(mp.project_l1(np.array([1.0, 1.0]), 1.0), [0.5, 0.5], atol=1e-12)
    np.testing.assert_allclose(mp.project_l2(np.array([3.0, 4.0]), 1.0), [0.6, 0.8], atol=1e-12)
    np.testing.assert_allclose(mp.project_linf(np.array([0.7, -1.2]), 1.0), [0.7, -1.0])
    x, budgets, z = mp.bilevel_project(np.eye(2), 1.0)
    np.testing.assert_allclose(x, 0.5 * np.eye(2), atol=1e-12)
    np.testing.assert_allclose(budgets, [0.5, 0.5], atol=1e-12)
    assert z == 0
    y = np.array([1.0, 0.2, 0.5, 0.4]).reshape(2, 1, 2)
    x = mp.multilevel_project(y, "inf,inf,1", 1.0)
    np.testing.assert_allclose(x, np.array([0.8, 0.2, 0.5, 0.2]).reshape(2, 1, 2), atol=1e-12)
    assert mp.multilevel_norm(x, "inf,inf,1") <= 1.0 + 1e-9
    assert mp.matrix_pq_norm(np.array([[1.0, 0.0], [1.0, 0.0]]), "1", "inf") == pytest.approx(1.0)
    assert mp.structured_sparsity(np.array([[1.0, 0.0], [1.0, 0.0]]), 0.0) == (1, 0.5)
    rng = np.random.default_rng(0)
    y = rng.normal(size=(30, 20))
    x, budgets, _ = mp.bilevel_project(y, 2.0)
    assert mp.matrix_pq_norm(x, "1", "inf") <= 2.0 * (1 + 1e-9)
    with pytest.raises(ValueError):
        mp.project_l1(np.array([1.0]), -1.0)
    with pytest.raises(ValueError):
        mp.multilevel_project(np.eye(2), "inf,bogus", 1.0)


def test_nonfinite_is_value_error():
    y = np.ones((5, 7), np.float32)
    for bad in (np.nan, np.inf, -np.inf):
        for q in NORMS:
            y2 = y.copy()
            y2[3, 4] = bad
            with pytest.raises(mp.MpValueError):
                mp.bilevel_project(y2, 1.0, "1", q)
    t = np.ones((3, 4, 5))
    t[1, 2, 3] = np.nan
    with pytest.raises(mp.MpValueError):
        mp.multilevel_project(t, "inf,inf,1", 1.0)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("n,m", [(600, 24), (1500, 16), (3000, 8), (4096, 64)])
def test_nonfinite_on_l1_strip_routes(dt, n, m):
    """Non-finite input on the TMA / hybrid l1 strip routes: every CTA leaves
    early with its strip copies drained; the call reports ValueError, and the
    next call on the same context is clean."""
    y = datagen.normal(5, (n, m)).astype(dt)
    for bad in (np.nan, np.inf):
        y2 = y.copy()
        y2[n // 2, m - 1] = bad
        with pytest.raises(mp.MpValueError):
            mp.bilevel_project(y2, 1.0, "1", "1")
    eta = 0.05 * float(np.abs(y.astype(np.float64)).sum())
    x, _, _ = mp.bilevel_project(y, eta, "1", "1")
    ref = O.bilevel(y.astype(np.float64), eta, "1", "1")
    check_bilevel(x, y, ref, "1")


# ------------------------------------------------ configs (scaled, oracle)
@pytest.mark.parametrize("p,q", [("1", "inf"), ("1", "1"), ("1", "2"), ("2", "inf"), ("inf", "inf"), ("2", "1")])
@pytest.mark.parametrize("shape", [(1, 1), (1, 37), (37, 1), (129, 67), (300, 1001), (1000, 1000)])
def test_bilevel_parity_shapes(p, q, shape):
    y = datagen.normal(11, shape)
    for rel in (0.0, 0.02, 0.3, 1.2):
        eta = rel * O.matrix_pq_norm(y.astype(np.float64), p, q)
        ref = oracle_bilevel(y, eta, p, q)
        x, b, z = run(y, eta, p, q)
        check_bilevel(x, y, ref, q, zero_cols_gpu=z)
        if rel >= 1.2:
            assert bit_equal(x, y)  # feasible input is the identity, bit for bit


def test_config1_full():
    y = datagen.config_input(1)
    eta = 0.1 * O.matrix_pq_norm(y.astype(np.float64), "1", "inf")
    ref = oracle_bilevel(y, eta)
    x, b, z = run(y, eta)
    rep = check_bilevel(x, y, ref, "inf", zero_cols_gpu=z)
    assert z == ref["zero_columns"]
    assert rep["max_rel"] < 1e-6


@pytest.mark.parametrize("rel", [0.001, 0.01, 0.1, 0.5])
def test_config2_full_radius_sweep(rel):
    """Headline config: 10000 x 10000 U[-1,1], element-wise vs the oracle."""
    y = datagen.config_input(2)
    y64 = y.astype(np.float64)
    eta = rel * O.matrix_pq_norm(y64, "1", "inf")
    ref = O.bilevel(y64, eta)
    del y64
    x, b, z = run(y, eta)
    check_bilevel(x, y, ref, "inf", zero_cols_gpu=z)
    np.testing.assert_allclose(b, ref["budgets"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("q", ["1", "2"])
def test_config3_full(q):
    y = datagen.config_input(3)
    y64 = y.astype(np.float64)
    eta = 0.05 * O.matrix_pq_norm(y64, "1", q)
    ref = O.bilevel(y64, eta, "1", q)
    del y64
    x, b, z = run(y, eta, "1", q)
    check_bilevel(x, y, ref, q, zero_cols_gpu=z)


def test_config4_full_trilevel():
    t = datagen.config_input(4)
    t64 = t.astype(np.float64)
    eta = 0.05 * O.multilevel_norm(t64, ["inf", "inf", "1"])
    xr = O.multilevel(t64, ["inf", "inf", "1"], eta)
    x = mp.trilevel_project_l1infinf(t, eta)
    assert x.dtype == np.float32
    # tri-level == bi-level on the (d0*d1, d2) reshape
    ref = O.bilevel(t64.reshape(256 * 256, 256), eta)
    assert np.array_equal(ref["X"].reshape(t.shape), xr)
    check_bilevel(x.reshape(256 * 256, 256), t.reshape(256 * 256, 256), ref, "inf")


def _ref_bilevel_dict(y64, eta, p, q):
    """The compiled, unmodified reference (oracle/_ref) in the dict shape
    check_bilevel reads: X, budgets, zero_columns, plus the column norms and
    the outer l1 threshold recovered from its budgets."""
    r = O.ref_bilevel(y64, eta, p, q, workers=os.cpu_count() or 1)
    a = np.abs(y64)
    v = a.sum(0) if q == "1" else (np.sqrt((a * a).sum(0)) if q == "2" else a.max(0))
    tau = -1.0
    if p == "1" and np.any(r["budgets"] > 0) and v.sum() > eta:
        tau = float(np.max(np.where(r["budgets"] > 0, v - r["budgets"], -np.inf)))
    return {"X": r["X"], "budgets": r["budgets"], "zero_columns": r["zero_columns"], "v": v, "tau": tau}


@pytest.mark.parametrize("case", ["c2_r0.1", "c3_l11", "c3_l12", "c4"])
def test_config_scale_against_compiled_reference(case):
    """Full-size parity directly against the compiled reference library (not
    the C restatement): config 2 at one radius, config 3 l1,1 / l1,2, config 4."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    if case == "c4":
        t = datagen.config_input(4)
        t64 = t.astype(np.float64)
        eta = 0.05 * O.ref_multilevel_norm(t64, ["inf", "inf", "1"])
        xr, chain_r = O.ref_multilevel(t64, ["inf", "inf", "1"], eta, want_chain=True)
        x, chain = mp.multilevel_project(t, "inf,inf,1", eta, return_chain=True)
        check_multilevel(x, t, [2, 2, 0], xr, chain_r, chain)
        return
    cfg, p, q, rel = {"c2_r0.1": (2, "1", "inf", 0.1), "c3_l11": (3, "1", "1", 0.05),
                      "c3_l12": (3, "1", "2", 0.05)}[case]
    y = datagen.config_input(cfg)
    y64 = y.astype(np.float64)
    eta = rel * O.ref_multilevel_norm(y64, [q, p])
    ref = _ref_bilevel_dict(y64, eta, p, q)
    del y64
    x, b, z = run(y, eta, p, q)
    check_bilevel(x, y, ref, q, zero_cols_gpu=z)
    assert z == ref["zero_columns"]


def test_config5_iteration0_full():
    y = datagen.config_input(5)
    v = np.abs(y).max(axis=0).astype(np.float64)
    eta = datagen.config5_eta(v)
    y64 = y.astype(np.float64)
    ref = O.bilevel(y64, eta)
    del y64
    x, b, z = run(y, eta)
    check_bilevel(x, y, ref, "inf", zero_cols_gpu=z)
    assert ref["zero_columns"] == 7373 and z == 7373


# --------------------------------------------------------- edge cases
def test_ragged_and_unaligned():
    rng = np.random.default_rng(3)
    for n, m in [(5, 3), (7, 5), (64, 6), (33, 1023), (2, 4097)]:
        y = rng.normal(size=(n, m)).astype(np.float32)
        for q in NORMS:
            eta = 0.2 * O.matrix_pq_norm(y.astype(np.float64), "1", q)
            x, b, z = run(y, eta, "1", q)
            check_bilevel(x, y, oracle_bilevel(y, eta, "1", q), q, zero_cols_gpu=z)


@pytest.mark.parametrize("m", [2049, 9999, 16384, 24576, 70000, 130000])
def test_wide_outer_cluster_and_cooperative(m):
    """K2: one CTA (registers, or shared memory up to m = 24576), 1..16-CTA
    clusters (m <= 98304) and a cooperative grid beyond."""
    y = datagen.normal(12, (3, m))
    for q in NORMS:
        eta = 0.05 * O.matrix_pq_norm(y.astype(np.float64), "1", q)
        x, b, z = run(y, eta, "1", q)
        check_bilevel(x, y, oracle_bilevel(y, eta, "1", q), q, zero_cols_gpu=z)


def test_large_vector_ball():
    v = datagen.normal(13, (300001,)).astype(np.float64)
    for q in NORMS:
        r = 0.1 * O.multilevel_norm(v, [q])
        np.testing.assert_allclose(mp.project_ball(v, q, r), O.project_ball(v, q, r), rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("n,m", [(1000, 64), (2000, 48), (4096, 24), (8000, 12), (8193, 8), (3000, 6), (1, 32),
                                 (7, 4), (4095, 40), (513, 24), (1025, 32), (2049, 16), (4097, 8)])
def test_l11_register_and_staged_geometries(dt, n, m):
    """Every K3b l1 route: register strips of 16P-byte row pieces (P = 8, 4,
    2, 1 by n), the TMA strips at their row-count boundaries (128 threads:
    513 / 1025..2048 rows; 256: 2049..4096; f64 512: 4097..8192), the
    shared-memory quad strip (n > 8192) and the column kernels (m not a
    multiple of 4); mixed column scales so strips hold zeroed, projected and
    (p = 2) shrunk columns; tie-heavy integer data."""
    rng = np.random.default_rng(n * 7 + m)
    scale = np.exp(rng.normal(size=m) * 1.5)
    for kind in ("normal", "ties"):
        if kind == "normal":
            y = (rng.normal(size=(n, m)) * scale).astype(dt)
        else:
            y = (rng.integers(-3, 4, size=(n, m)) * np.round(scale * 4)).astype(dt)
        for p, rel in (("1", 0.05), ("1", 0.3), ("2", 0.5)):
            eta = rel * O.matrix_pq_norm(y.astype(np.float64), p, "1")
            x, b, z = run(y, eta, p, "1")
            check_bilevel(x, y, oracle_bilevel(y, eta, p, "1"), "1", zero_cols_gpu=z)


def test_l11_unstaged_tall_columns():
    """n beyond the cluster's shared-memory capacity: unstaged strip path."""
    y = datagen.normal(14, (60000, 40))
    eta = 0.05 * O.matrix_pq_norm(y.astype(np.float64), "1", "1")
    x, b, z = run(y, eta, "1", "1")
    check_bilevel(x, y, oracle_bilevel(y, eta, "1", "1"), "1", zero_cols_gpu=z)


def test_eta_zero_and_zero_sign():
    y = datagen.normal(15, (50, 40))
    x, b, z = run(y, 0.0)
    assert z == 40 and np.all(x == 0)
    # default: zero-budget columns written as +0 without a read
    assert not np.any(np.signbit(x))
    # exact flag: copysign(0, y) bytes like proj/src/fiber_kernels.cpp:47
    x2, _, _ = run(y, 0.0, flags=mp.MP_FLAG_EXACT_ZERO_SIGN)
    ref = oracle_bilevel(y, 0.0)
    assert bit_equal(x2, ref["X"].astype(np.float32))


def test_exact_flag_bitwise_vs_rounded_reference():
    """With exact zero signs, l_{1,inf} output equals RN(reference) bit for
    bit except in the near-threshold band (compare uses RD(u), value RN(u))."""
    y = datagen.uniform(16, (400, 333), -1.0, 1.0)
    eta = 0.05 * O.matrix_pq_norm(y.astype(np.float64), "1", "inf")
    ref = oracle_bilevel(y, eta)
    x, _, _ = run(y, eta, flags=mp.MP_FLAG_EXACT_ZERO_SIGN)
    near = np.abs(ref["v"] - ref["tau"]) <= 1e-5 * ref["tau"]
    same = np.all(x.view(np.uint32) == ref["X"].astype(np.float32).view(np.uint32), axis=0)
    assert np.all(same | near)


# ------------------------------------------------------ device API / graphs
def test_device_api_graph_determinism_inplace():
    import torch
    y = torch.from_numpy(datagen.uniform(17, (2000, 3000), -1.0, 1.0)).cuda()
    eta = 0.01 * float(y.abs().amax(dim=0).double().sum())
    proj = mp.BilevelProjector(2000, 3000, "float32", "1", "inf")
    x1 = torch.empty_like(y)
    proj(y, x1, eta)
    torch.cuda.synchronize()
    x2 = torch.empty_like(y)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            proj(y, x2, eta, stream=s)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(x1.view(torch.int32), x2.view(torch.int32))
    y3 = y.clone()
    proj(y3, y3, eta)  # in place
    torch.cuda.synchronize()
    assert torch.equal(x1.view(torch.int32), y3.view(torch.int32))
    for q in ("1", "2"):
        pq = mp.BilevelProjector(2000, 3000, "float32", "1", q)
        a, b = torch.empty_like(y), torch.empty_like(y)
        pq(y, a, eta * 50)
        pq(y, b, eta * 50)
        torch.cuda.synchronize()
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))  # run-to-run bitwise


@pytest.mark.parametrize("n,m,dt", [(4096, 1024, "float32"), (3000, 512, "float32"), (4096, 256, "float64"),
                                    (6000, 128, "float64")])
def test_l11_inplace_on_split_apply_strips(n, m, dt):
    """l1,1 in place (x is y) on the 256 / 512-thread TMA strips, whose apply
    rewrites the register pieces in place and reloads them for the next
    strip: same bytes as out of place, and parity with the oracle."""
    import torch
    rng = np.random.default_rng(n + m)
    scale = np.exp(rng.normal(size=m))  # zeroed, projected and feasible columns
    y_h = (rng.normal(size=(n, m)) * scale).astype(dt)
    y = torch.from_numpy(y_h).cuda()
    eta = 0.2 * O.matrix_pq_norm(y_h.astype(np.float64), "1", "1")
    proj = mp.BilevelProjector(n, m, dt, "1", "1")
    x = torch.empty_like(y)
    proj(y, x, eta)
    z = proj.info().zero_columns
    y2 = y.clone()
    proj(y2, y2, eta)
    torch.cuda.synchronize()
    it = torch.int32 if dt == "float32" else torch.int64
    assert torch.equal(x.view(it), y2.view(it))
    check_bilevel(x.cpu().numpy(), y_h, oracle_bilevel(y_h, eta, "1", "1"), "1", zero_cols_gpu=z)


def test_idempotence_full_size():
    """Project, then project the result at eta(1+1e-6): identical bytes."""
    y = datagen.config_input(2, scale=0.5)
    eta = 0.01 * O.matrix_pq_norm(y.astype(np.float64), "1", "inf")
    x, _, _ = run(y, eta)
    x2, _, _ = run(x, eta * (1 + 1e-6))
    assert bit_equal(x, x2)
    colmax = np.abs(x.astype(np.float64)).max(axis=0)
    assert colmax.sum() <= eta * (1 + 1e-6)


def test_config5_loop_sampled_parity():
    """Config 5: 32768 x 8192 Laplace(0, 0.01), eta zeroing ~90% of columns at
    iteration 0, projected 100 times with a seeded N(0, 1e-4^2) perturbation
    between calls (device Philox).  Iterations 0, 1, 49 and 99 are checked
    element-wise against the oracle on the GPU's own perturbed input
    (SURVEY.md §8d); the zeroed fraction must drift down (§0.8)."""
    import torch
    y = datagen.config_input(5)
    eta = datagen.config5_eta(np.abs(y).max(axis=0).astype(np.float64))
    x = torch.from_numpy(y).cuda()
    proj = mp.BilevelProjector(*y.shape)
    zeros, checked = [], 0
    for t in range(100):
        if t > 0:
            mp.perturb_gaussian(x, 1e-4, seed=6, iteration=t)
        sample = t in (0, 1, 49, 99)
        if sample:
            x_in = x.cpu().numpy()
        proj(x, x, eta)
        torch.cuda.synchronize()
        info = proj.info()
        zeros.append(int(info.zero_columns))
        if sample:
            ref = O.bilevel(x_in.astype(np.float64), eta)
            check_bilevel(x.cpu().numpy(), x_in, ref, "inf", zero_cols_gpu=info.zero_columns)
            checked += 1
            del x_in, ref
    assert checked == 4
    assert zeros[0] == 7373
    assert zeros[-1] < zeros[0]  # the zeroed set shrinks under the perturbation


def test_perturbation_is_seeded_gaussian():
    import torch
    a = torch.zeros(1 << 20, device="cuda")
    b = torch.zeros(1 << 20, device="cuda")
    mp.perturb_gaussian(a, 1.0, seed=6, iteration=3)
    mp.perturb_gaussian(b, 1.0, seed=6, iteration=3)
    assert torch.equal(a, b)  # stateless and reproducible
    c = torch.zeros(1 << 20, device="cuda")
    mp.perturb_gaussian(c, 1.0, seed=6, iteration=4)
    assert not torch.equal(a, c)
    m, s = float(a.mean()), float(a.std())
    assert abs(m) < 5e-3 and abs(s - 1.0) < 5e-3


def test_radius_sweep_host_api_matches_single_calls():
    y = datagen.uniform(21, (3000, 2000), -1.0, 1.0)
    colsum = float(np.abs(y).max(axis=0).astype(np.float64).sum())
    etas = [0.001 * colsum, 0.1 * colsum, 0.5 * colsum, 2.0 * colsum, 0.0]
    res = mp.bilevel_radius_sweep(y, etas)
    for (x, b, z), e in zip(res, etas):
        x1, b1, z1 = mp.bilevel_project(y, e)
        assert bit_equal(x, x1) and z == z1
        np.testing.assert_array_equal(np.asarray(b), np.asarray(b1))


@pytest.mark.parametrize("q", ["inf", "2", "1"])
def test_beyond_int32_element_count(q):
    """40000 x 60000 (8192 x 300000 for l1,1) fp32, 2.4-2.5e9 elements
    (> 2^31): 64-bit offsets end to end.
    Inputs are generated on the device (torch); the checker is the oracle's
    outer projection of exact column norms (torch.amax / float64 sums) and the
    per-column apply on sampled columns."""
    import torch
    n, m = (8192, 300000) if q == "1" else (40000, 60000)
    g = torch.Generator(device="cuda").manual_seed(11)
    y = torch.rand((n, m), generator=g, device="cuda", dtype=torch.float32).mul_(2).sub_(1)
    if q == "inf":
        v = y.abs().amax(dim=0).double().cpu().numpy()
    elif q == "2":
        v = torch.linalg.vector_norm(y.double(), dim=0).cpu().numpy()
    else:
        v = y.double().abs().sum(dim=0).cpu().numpy()
    eta = 0.05 * float(v.sum())
    proj = mp.BilevelProjector(n, m, "float32", "1", q)
    x = proj(y, torch.empty_like(y), eta)
    torch.cuda.synchronize()
    inf = proj.info()
    assert inf.status == 0
    u_ref = O.project_ball(v, "1", eta)
    u_gpu = proj.budgets.cpu().numpy()
    np.testing.assert_allclose(u_gpu, u_ref, rtol=1e-9, atol=1e-12)
    rng = np.random.default_rng(5)
    cols = np.concatenate([[0, m - 1], rng.choice(m, 30, replace=False)])
    yc = y[:, cols].double().cpu().numpy()
    xc = x[:, cols].double().cpu().numpy()
    ref = O.project_fibers(yc, q, v[cols], u_ref[cols])
    if q == "1":
        check_bilevel(xc, yc, {"X": ref, "v": v[cols], "tau": -1.0, "zero_columns": 0}, "1")
    else:
        np.testing.assert_allclose(xc, ref, rtol=1e-6, atol=1e-7)
    del y, x
    torch.cuda.empty_cache()


def test_async_sweeps_pipeline_equals_synchronous():
    """mp_bilevel_sweep_host_async: several sweeps in flight on one context
    (including a third issued without a wait) give the synchronous results."""
    import ctypes as C
    from paper_2405_02086_b200 import _capi
    lib = _capi.lib()
    rng = np.random.default_rng(9)
    n, m = 300, 700
    ys = [rng.normal(size=(n, m)).astype(np.float32) for _ in range(4)]
    etas = np.ascontiguousarray([0.01, 0.2, 0.6], np.float64) * float(np.abs(ys[0]).max(axis=0).sum())
    ref = [mp.bilevel_radius_sweep(y, etas) for y in ys]
    ctx = lib.mp_context_create(0)
    outs = [[np.empty_like(ys[0]) for _ in etas] for _ in ys]
    zeros = [np.empty(len(etas), np.int64) for _ in ys]
    buds = [np.empty((len(etas), m)) for _ in ys]
    tks = []
    for i, y in enumerate(ys):
        ptrs = (C.c_void_p * len(etas))(*[C.c_void_p(o.ctypes.data) for o in outs[i]])
        tk = C.c_uint64()
        _capi.check(lib.mp_bilevel_sweep_host_async(ctx, y.ctypes.data, ptrs, _capi.MP_F32, n, m, 0, 2,
                                                    etas.ctypes.data, len(etas), buds[i].ctypes.data,
                                                    zeros[i].ctypes.data, 0, C.byref(tk)))
        tks.append(tk.value)
        if i == 1:
            _capi.check(lib.mp_context_wait(ctx, tks[0]))
    for tk in tks:
        _capi.check(lib.mp_context_wait(ctx, tk))
    lib.mp_context_destroy(ctx)
    for i in range(len(ys)):
        for k in range(len(etas)):
            xr, br, zr = ref[i][k]
            assert bit_equal(outs[i][k], xr)
            assert np.array_equal(buds[i][k], np.asarray(br)) and zeros[i][k] == zr
