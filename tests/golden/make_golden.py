"""Generate tests/golden/golden.npz from the UNMODIFIED reference library.

Run in the build container, where /root/reference exists and oracle/Makefile
has compiled oracle/_ref/libmultiproj_ref.so from the reference sources:

    python tests/golden/make_golden.py

The fixtures are small seeded cases (inputs are fp32-representable so the
fp32 device path consumes exactly the same values) covering every
(p, q) pair, eta = 0, feasible inputs, ties, zero columns, ragged shapes and
multi-level specs of order 1-4, and the exact Euclidean l1,inf projection.
Outputs are the reference's own f64 results.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

NORMS = ["1", "2", "inf"]


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def main():
    assert O.ref_available(), "build oracle/_ref first (make -C oracle ref)"
    rng = np.random.default_rng(2405_02086)
    out = {}
    # ---- bilevel
    cases = []
    for p in NORMS:
        for q in NORMS:
            for shape in [(1, 1), (2, 2), (3, 7), (17, 5), (40, 24), (33, 130)]:
                rels = [0.0, 0.03, 0.3, 0.9, 1.5] if shape[0] * shape[1] < 1000 else [0.05, 0.6]
                for rel in rels:
                    y = f32(rng.normal(size=shape))
                    if rng.uniform() < 0.3:  # some zero columns and exact ties
                        y[:, rng.integers(0, shape[1])] = 0.0
                        y[rng.integers(0, shape[0]), :] = y[0, 0]
                    cases.append((p, q, y, rel))
    for i, (p, q, y, rel) in enumerate(cases):
        eta = rel * O.ref_multilevel_norm(y, [q, p])
        r = O.ref_bilevel(y, eta, p, q)
        out[f"bi{i}_y"] = y.astype(np.float32)
        out[f"bi{i}_meta"] = np.array([O.NORMS[p], O.NORMS[q], eta], np.float64)
        out[f"bi{i}_x"] = r["X"]
        out[f"bi{i}_b"] = r["budgets"]
        out[f"bi{i}_z"] = np.array([r["zero_columns"]], np.int64)
    out["bi_count"] = np.array([len(cases)])
    # ---- multilevel (iterative form, with budget chain)
    mcases = []
    for order in [1, 2, 3, 4]:
        for _ in range(8):
            shape = tuple(int(s) for s in rng.integers(1, 7, order))
            lv = [NORMS[int(k)] for k in rng.integers(0, 3, order)]
            if rng.uniform() < 0.5:
                lv[-1] = "1"
            t = f32(rng.uniform(-1, 1, shape))
            rel = float(rng.choice([0.0, 0.1, 0.5, 0.95, 2.0]))
            mcases.append((t, lv, rel))
    mcases.append((f32(rng.normal(size=(8, 8, 8))), ["inf", "inf", "1"], 0.05))
    for i, (t, lv, rel) in enumerate(mcases):
        eta = rel * O.ref_multilevel_norm(t, lv)
        x, chain = O.ref_multilevel(t, lv, eta, want_chain=True)
        out[f"ml{i}_t"] = t.astype(np.float32)
        out[f"ml{i}_lv"] = np.array([O.NORMS[q] for q in lv], np.int32)
        out[f"ml{i}_eta"] = np.array([eta])
        out[f"ml{i}_x"] = x
        out[f"ml{i}_chain"] = np.concatenate([c.reshape(-1) for c in chain]) if chain else np.zeros(0)
    out["ml_count"] = np.array([len(mcases)])
    # ---- vector balls (sort and fast paths agree)
    vcases = []
    for q in NORMS:
        for n in [1, 2, 5, 100, 4097]:
            y = f32(rng.normal(size=n))
            for rel in [0.0, 0.2, 0.7, 1.3]:
                vcases.append((q, y, rel))
    for i, (q, y, rel) in enumerate(vcases):
        r = rel * np.abs(y).sum() if q == "1" else rel * (np.sqrt((y * y).sum()) if q == "2" else np.abs(y).max())
        out[f"vb{i}_y"] = y.astype(np.float32)
        out[f"vb{i}_meta"] = np.array([O.NORMS[q], r])
        out[f"vb{i}_x"] = O.ref_project_ball(y, q, r)
    out["vb_count"] = np.array([len(vcases)])
    # ---- generator stream (datagen must restate the reference RNG exactly)
    out["rng_raw_seed7"] = O.ref_gen_raw(7, 64)
    out["rng_uniform_seed2"] = O.ref_gen_uniform(2, 64, -1.0, 1.0)
    out["rng_normal_seed1"] = O.ref_gen_normal(1, 64)
    # ---- exact Euclidean l1,inf (proj/src/euclidean.cpp), worked examples of
    # proj/tests/test_euclidean.cpp:20-48 first
    ecases = [(f32([[1, 0.5], [1, 0]]), 1.0, None), (f32([[0.3, 0.1], [-0.2, 0.05]]), 2.0, None),
              (f32([[1, 2], [3, 4]]), 0.0, None)]
    for shape in [(1, 1), (2, 3), (5, 1), (4, 4), (9, 7), (40, 24), (33, 130), (300, 17)]:
        for rel in [0.0, 0.05, 0.3, 0.7, 0.99, 1.2]:
            y = f32(rng.normal(size=shape))
            if rng.uniform() < 0.3:  # ties and zero columns
                y = f32(np.round(y * 2) / 2)
                y[:, rng.integers(0, shape[1])] = 0.0
            ecases.append((y, None, rel))
    for i, (y, eta, rel) in enumerate(ecases):
        if eta is None:
            eta = rel * float(np.abs(y).max(axis=0).sum())
        x, b, th = O.ref_euclid(y, eta)
        out[f"eu{i}_y"] = y.astype(np.float32)
        out[f"eu{i}_eta"] = np.array([eta])
        out[f"eu{i}_x"] = x
        out[f"eu{i}_b"] = b
        out[f"eu{i}_theta"] = np.array([th])
    out["eu_count"] = np.array([len(ecases)])
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(cases)} bilevel, {len(mcases)} multilevel, {len(vcases)} vector, "
          f"{len(ecases)} euclid cases, "
          f"{os.path.getsize(path) / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
