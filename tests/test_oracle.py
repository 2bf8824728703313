"""Pin the CPU oracle (oracle/mp_oracle.c) before trusting it as the checker.

1. The reference's own known answers (worked examples from its tests).
2. The golden fixtures produced by the compiled reference
   (tests/golden/make_golden.py) -- bit-exact.
3. Bit-exact agreement with the compiled reference on fresh random inputs
   (when oracle/_ref was built in this container).
"""
import numpy as np
import pytest

from oracle import oracle as O

bit_equal = lambda a, b: np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


# ------------------------------------------------------------ known answers
def test_bilevel_identity_matrix():  # proj/tests/test_bilevel.cpp:11-19
    r = O.bilevel(np.array([[1.0, 0.0], [0.0, 1.0]]), 1.0)
    np.testing.assert_allclose(r["budgets"], [0.5, 0.5], rtol=1e-12)
    np.testing.assert_allclose(r["X"].reshape(-1), [0.5, 0, 0, 0.5], atol=1e-12)
    assert r["zero_columns"] == 0


def test_bilevel_zeroes_weak_column():  # proj/tests/test_bilevel.cpp:21-31
    r = O.bilevel(np.array([[0.9, 0.1], [0.1, 0.05]]), 0.6)
    np.testing.assert_allclose(r["budgets"], [0.6, 0.0], atol=1e-12)
    np.testing.assert_allclose(r["X"].reshape(-1), [0.6, 0, 0.1, 0], atol=1e-12)
    assert r["zero_columns"] == 1


def test_bilevel_l11_worked_example():  # proj/tests/test_bilevel.cpp:33-40
    r = O.bilevel(np.array([[0.5, 0.25], [0.5, 0.25]]), 1.0, "1", "1")
    np.testing.assert_allclose(r["budgets"], [0.75, 0.25], rtol=1e-12)
    np.testing.assert_allclose(r["X"].reshape(-1), [0.375, 0.125, 0.375, 0.125], atol=1e-12)


def test_bilevel_l12_worked_example():  # proj/tests/test_bilevel.cpp:42-49
    r = O.bilevel(np.array([[3.0, 0.0], [4.0, 0.0]]), 1.0, "1", "2")
    np.testing.assert_allclose(r["budgets"], [1.0, 0.0], atol=1e-12)
    np.testing.assert_allclose(r["X"].reshape(-1), [0.6, 0, 0.8, 0], atol=1e-12)


def test_bilevel_errors():  # proj/tests/test_bilevel.cpp:51-56
    with pytest.raises(O.OracleError) as e:
        O.bilevel(np.eye(2), -1.0)
    assert e.value.code == 1
    with pytest.raises(O.OracleError) as e:
        O.bilevel(np.array([1.0, 2.0, 3.0]), 1.0)
    assert e.value.code == 2


def test_bilevel_feasible_identity():  # proj/tests/test_bilevel.cpp:86-91
    y = np.array([[0.1, -0.2, 0.05], [0.0, 0.1, 0.02]])
    norm = O.matrix_pq_norm(y, "1", "inf")
    assert bit_equal(O.bilevel(y, norm + 1.0)["X"], y)


def test_trilevel_worked_example():  # proj/tests/test_multilevel.cpp:21-29
    y = np.array([1.0, 0.2, 0.5, 0.4]).reshape(2, 1, 2)
    x = O.multilevel(y, ["inf", "inf", "1"], 1.0)
    np.testing.assert_allclose(x.reshape(-1), [0.8, 0.2, 0.5, 0.2], atol=1e-12)
    assert O.multilevel_norm(x, ["inf", "inf", "1"]) == pytest.approx(1.0, rel=1e-12)


def test_multilevel_norm_example():  # proj/tests/test_multilevel.cpp:77-82
    y = np.array([1.0, 0.2, 0.5, 0.4]).reshape(2, 1, 2)
    assert O.multilevel_norm(y, ["inf", "inf", "1"]) == pytest.approx(1.4, rel=1e-12)


def test_l1_worked_examples():  # proj/tests/test_vector_balls.cpp:30-47
    np.testing.assert_allclose(O.project_l1([1.0, 1.0], 1.0)[0], [0.5, 0.5], atol=1e-12)
    np.testing.assert_allclose(O.project_l1([0.9, 0.1], 0.6)[0], [0.6, 0.0], atol=1e-12)
    np.testing.assert_allclose(O.project_ball([3.0, 4.0], "2", 1.0), [0.6, 0.8], atol=1e-12)
    np.testing.assert_allclose(O.project_ball([0.7, -1.2], "inf", 1.0), [0.7, -1.0])


def test_random_invariants():  # proj/tests/test_bilevel.cpp:58-84
    rng = np.random.default_rng(21)
    for _ in range(200):
        n, m = rng.integers(1, 13, 2)
        y = rng.uniform(-1, 1, (n, m))
        eta = rng.uniform() * 1.2 * O.matrix_pq_norm(y, "1", "inf")
        r = O.bilevel(y, eta)
        assert O.matrix_pq_norm(r["X"], "1", "inf") <= eta * (1 + 1e-9) + 1e-15
        assert np.all(np.abs(r["X"]).max(axis=0) <= r["budgets"] * (1 + 1e-9) + 1e-15)
        assert r["zero_columns"] == O.structured_sparsity(r["X"], 0.0)
        assert bit_equal(O.bilevel(r["X"], eta * (1 + 1e-9))["X"], r["X"])


def test_fast_equals_sort():  # proj/tests/test_vector_balls.cpp:58-73
    rng = np.random.default_rng(5)
    for _ in range(300):
        y = rng.normal(size=int(rng.integers(1, 200)))
        r = rng.uniform() * np.abs(y).sum()
        a, ta, ka = O.project_l1(y, r)
        b, tb, kb = O.project_l1(y, r, sort=True)
        assert bit_equal(a, b) and ta == tb and ka == kb


# ------------------------------------------------------------ golden vectors
def test_golden_bilevel(golden):
    for i in range(int(golden["bi_count"][0])):
        y = golden[f"bi{i}_y"].astype(np.float64)
        p, q, eta = golden[f"bi{i}_meta"]
        r = O.bilevel(y, eta, int(p), int(q))
        assert bit_equal(r["X"], golden[f"bi{i}_x"]), i
        assert bit_equal(r["budgets"], golden[f"bi{i}_b"]), i
        assert r["zero_columns"] == golden[f"bi{i}_z"][0], i


def test_golden_multilevel(golden):
    for i in range(int(golden["ml_count"][0])):
        t = golden[f"ml{i}_t"].astype(np.float64)
        lv = [int(k) for k in golden[f"ml{i}_lv"]]
        x, chain = O.multilevel(t, lv, float(golden[f"ml{i}_eta"][0]), want_chain=True)
        assert bit_equal(x, golden[f"ml{i}_x"]), i
        flat = np.concatenate([c.reshape(-1) for c in chain]) if chain else np.zeros(0)
        assert bit_equal(flat, golden[f"ml{i}_chain"]), i


def test_golden_vector_balls(golden):
    for i in range(int(golden["vb_count"][0])):
        y = golden[f"vb{i}_y"].astype(np.float64)
        q, r = golden[f"vb{i}_meta"]
        assert bit_equal(O.project_ball(y, int(q), r), golden[f"vb{i}_x"]), i


# --------------------------------------------- direct comparison with _ref
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_restatement_matches_reference_bilevel():
    rng = np.random.default_rng(77)
    for _ in range(300):
        n, m = (int(v) for v in rng.integers(1, 20, 2))
        y = rng.normal(size=(n, m))
        p, q = (["1", "2", "inf"][int(k)] for k in rng.integers(0, 3, 2))
        eta = rng.uniform() * 1.2 * O.matrix_pq_norm(y, p, q)
        a, b = O.bilevel(y, eta, p, q), O.ref_bilevel(y, eta, p, q, workers=int(rng.integers(1, 4)))
        assert bit_equal(a["X"], b["X"]) and bit_equal(a["budgets"], b["budgets"])
        assert a["zero_columns"] == b["zero_columns"]


@needs_ref
def test_restatement_matches_reference_multilevel():
    rng = np.random.default_rng(78)
    for _ in range(200):
        order = int(rng.integers(1, 5))
        shape = tuple(int(s) for s in rng.integers(1, 6, order))
        t = rng.uniform(-1, 1, shape)
        lv = [["1", "2", "inf"][int(k)] for k in rng.integers(0, 3, order)]
        eta = rng.uniform() * 1.2 * O.multilevel_norm(t, lv)
        x, ch = O.multilevel(t, lv, eta, want_chain=True)
        x2, ch2 = O.ref_multilevel(t, lv, eta, want_chain=True)
        assert bit_equal(x, x2)
        assert all(bit_equal(a, b) for a, b in zip(ch, ch2)) and len(ch) == len(ch2)
        # recursive == iterative (proj/tests/test_multilevel.cpp:44-67)
        assert bit_equal(O.ref_multilevel(t, lv, eta, recursive=True), x)


@needs_ref
def test_restatement_matches_reference_l1_large():
    rng = np.random.default_rng(79)
    y = rng.normal(size=100_000)  # proj/tests/test_vector_balls.cpp:58-73 (length 1e5)
    for rel in [0.01, 0.3, 0.9]:
        r = rel * np.abs(y).sum()
        assert bit_equal(O.project_l1(y, r)[0], O.ref_project_ball(y, "1", r))


@needs_ref
def test_trilevel_equals_reshaped_bilevel():
    rng = np.random.default_rng(80)
    for _ in range(50):
        d = rng.integers(1, 6, 3)
        t = rng.normal(size=tuple(int(v) for v in d))
        eta = rng.uniform() * O.multilevel_norm(t, ["inf", "inf", "1"])
        x = O.ref_trilevel(t, eta)
        xb = O.bilevel(t.reshape(int(d[0] * d[1]), int(d[2])), eta)["X"].reshape(t.shape)
        assert bit_equal(x, xb)
