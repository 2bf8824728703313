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


def test_golden_euclid(golden):  # proj/src/euclidean.cpp, fixtures from the compiled reference
    for i in range(int(golden["eu_count"][0])):
        y = golden[f"eu{i}_y"].astype(np.float64)
        x, b, th = O.euclid(y, float(golden[f"eu{i}_eta"][0]))
        assert bit_equal(x, golden[f"eu{i}_x"]), i
        assert bit_equal(b, golden[f"eu{i}_b"]), i
        assert th == golden[f"eu{i}_theta"][0], i


def test_euclid_worked_example():  # proj/tests/test_euclidean.cpp:20-34
    y = np.array([[1, 0.5], [1, 0]], float)
    x, b, th = O.euclid(y, 1.0)
    assert abs(th - 1 / 3) < 1e-12 and abs(b[0] - 5 / 6) < 1e-12 and abs(b[1] - 1 / 6) < 1e-12
    assert abs(((y - x) ** 2).sum() - 1 / 6) < 1e-12
    assert abs(((y - O.bilevel(y, 1.0)["X"]) ** 2).sum() - 0.1875) < 1e-12


def test_euclid_identity_zero_and_errors():  # proj/tests/test_euclidean.cpp:36-55
    y = np.array([[0.3, 0.1], [-0.2, 0.05]])
    x, b, th = O.euclid(y, 2.0)
    assert bit_equal(x, y) and th == 0.0
    x, b, th = O.euclid(np.array([[1.0, 2], [3, 4]]), 0.0)
    assert not x.any()
    with pytest.raises(O.OracleError):
        O.euclid(y, -1.0)


def test_euclid_kkt_and_never_worse_than_bilevel():  # proj/tests/test_euclidean.cpp:77-125
    rng = np.random.default_rng(43)
    for _ in range(100):
        n, m = (int(v) for v in rng.integers(2, 10, 2))
        y = rng.normal(size=(n, m))
        nrm = np.abs(y).max(axis=0).sum()
        eta = rng.uniform(0.05, 0.95) * nrm
        x, b, th = O.euclid(y, eta)
        assert th > 0.0
        resid = np.maximum(np.abs(y) - b[None, :], 0.0).sum(axis=0)
        act = b > 0
        np.testing.assert_allclose(resid[act], th, rtol=1e-9)
        assert np.all(resid[~act] <= th * (1 + 1e-9) + 1e-12)
        assert np.abs(x).max(axis=0).sum() <= eta * (1 + 1e-9) + 1e-15
        assert ((y - x) ** 2).sum() <= ((y - O.bilevel(y, eta)["X"]) ** 2).sum() + 1e-12


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


@needs_ref
def test_restatement_matches_reference_euclid():
    rng = np.random.default_rng(81)
    for _ in range(300):
        n, m = (int(v) for v in rng.integers(1, 14, 2))
        y = rng.normal(size=(n, m))
        if rng.uniform() < 0.3:
            y = np.round(y * 2) / 2  # ties
        eta = rng.uniform() * 1.2 * np.abs(y).max(axis=0).sum()
        a, b = O.euclid(y, eta), O.ref_euclid(y, eta)
        assert bit_equal(a[0], b[0]) and bit_equal(a[1], b[1]) and a[2] == b[2]


@needs_ref
def test_euclid_matches_budget_grid():  # proj/tests/test_euclidean.cpp:57-75
    rng = np.random.default_rng(41)
    for _ in range(30):
        n, m = int(rng.integers(1, 6)), int(rng.integers(1, 4))
        y = rng.uniform(-1, 1, (n, m))
        nrm = np.abs(y).max(axis=0).sum()
        eta = (0.2 + 0.7 * rng.uniform()) * nrm
        steps = 2000 if m == 3 else 10000
        x, b, th = O.euclid(y, eta)
        gb, _ = O.ref_budget_grid(y, eta, steps)
        assert ((y - x) ** 2).sum() <= O.ref_clip_cost(y, gb) + 1e-9
        assert abs(O.clip_cost(y, gb) - O.ref_clip_cost(y, gb)) <= 1e-15 * max(1.0, O.clip_cost(y, gb))
        assert np.all(np.abs(b - gb) <= 2 * eta / steps + 1e-9)
