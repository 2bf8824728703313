"""Randomised parity sweep: many small bi-level / multi-level / euclid / ball
projections with adversarial data (zero columns, ties, mixed magnitudes,
subnormal-free tiny and large scales, radii at 0, near the norm and above it)
against the oracle with the §8(c) rule."""
import numpy as np
import pytest

import paper_2405_02086_b200 as mp
from oracle import oracle as O
from tests.parity import check_bilevel

pytestmark = pytest.mark.gpu
NORMS = ["1", "2", "inf"]


def adversarial(rng, n, m, dt):
    kind = rng.integers(0, 6)
    if kind == 0:
        y = rng.normal(size=(n, m))
    elif kind == 1:  # heavy ties
        y = rng.integers(-2, 3, size=(n, m)).astype(float)
    elif kind == 2:  # mixed column scales
        y = rng.normal(size=(n, m)) * np.exp(rng.normal(size=m) * 3)
    elif kind == 3:  # sparse with zero columns
        y = rng.normal(size=(n, m)) * (rng.random((n, m)) < 0.2)
        y[:, rng.random(m) < 0.3] = 0.0
    elif kind == 4:  # tiny / large magnitudes
        y = rng.normal(size=(n, m)) * (1e-20 if rng.random() < 0.5 else 1e15)
    else:  # all equal magnitudes, random signs
        y = np.where(rng.random((n, m)) < 0.5, -1.0, 1.0) * 0.75
    return y.astype(dt)


@pytest.mark.parametrize("seed", range(8))
def test_bilevel_fuzz(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(40):
        # log-uniform shapes up to 2M elements: every K1 / K2 / K3 / K3b route
        n = int(np.exp(rng.uniform(0, np.log(20000))))
        m = int(np.exp(rng.uniform(0, np.log(30000))))
        if n * m > 2_000_000:
            m = max(1, 2_000_000 // n)
        dt = np.float32 if rng.random() < 0.6 else np.float64
        y = adversarial(rng, n, m, dt)
        p, q = NORMS[rng.integers(0, 3)], NORMS[rng.integers(0, 3)]
        nrm = O.matrix_pq_norm(y.astype(np.float64), p, q)
        eta = float(rng.choice([0.0, 1e-3, 0.1, 0.5, 0.999, 1.0, 1.7])) * nrm
        x, b, z = mp.bilevel_project(y, eta, p, q)
        ref = O.bilevel(y.astype(np.float64), eta, p, q)
        check_bilevel(x, y, ref, q, zero_cols_gpu=z)


@pytest.mark.parametrize("seed", range(4))
def test_multilevel_and_ball_fuzz(seed):
    rng = np.random.default_rng(2000 + seed)
    for _ in range(20):
        order = int(rng.integers(1, 5))
        shape = tuple(int(s) for s in rng.integers(1, 9, order))
        lv = [NORMS[k] for k in rng.integers(0, 3, order)]
        t = rng.normal(size=shape) * (rng.random(shape) < 0.7)
        eta = float(rng.choice([0.0, 0.05, 0.5, 1.2])) * O.multilevel_norm(t, lv)
        x = mp.multilevel_project(t, ",".join(lv), eta)
        xr = O.multilevel(t, lv, eta)
        np.testing.assert_allclose(x, xr, rtol=1e-9, atol=1e-12 * max(1.0, np.abs(xr).max(initial=0.0)))
    for _ in range(20):
        v = rng.normal(size=int(rng.integers(1, 5000))) * np.exp(rng.normal() * 3)
        q = NORMS[rng.integers(0, 3)]
        r = float(rng.choice([0.0, 0.01, 0.5, 2.0])) * O.multilevel_norm(v, [q])
        np.testing.assert_allclose(mp.project_ball(v, q, r), O.project_ball(v, q, r), rtol=1e-10,
                                   atol=1e-13 * max(1.0, np.abs(v).max()))


@pytest.mark.parametrize("seed", range(3))
def test_euclid_fuzz(seed):
    rng = np.random.default_rng(3000 + seed)
    for _ in range(15):
        n, m = int(rng.integers(1, 300)), int(rng.integers(1, 200))
        y = adversarial(rng, n, m, np.float64)
        nrm = float(np.abs(y).max(axis=0).sum())
        eta = float(rng.choice([0.0, 1e-3, 0.3, 0.9, 1.5])) * nrm
        x, b, th = mp.euclid_project_l1inf(y, eta)
        xr, br, tr = O.euclid(y, eta)
        np.testing.assert_allclose(th, tr, rtol=1e-10, atol=1e-300)
        np.testing.assert_allclose(b, br, rtol=1e-10, atol=1e-12 * max(1.0, nrm))
        np.testing.assert_allclose(x, xr, rtol=1e-10, atol=1e-12 * max(1.0, nrm))
