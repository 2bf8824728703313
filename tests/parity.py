"""Parity rule between the CUDA path and the CPU oracle.

Inputs are identical (fp32 values, upcast exactly to f64 for the oracle).
With rtol = 1e-5 (the north_star tolerance for fp32 output):

1. tau: |tau_gpu - tau_ref| <= rtol * tau_ref.
2. Near-threshold columns N = {j : |v_j - tau_ref| <= rtol * tau_ref}.
3. Zeroed-column sets may differ only inside N.
4. Elements of columns outside N: |x_gpu - x_ref| <= rtol * |x_ref| (+-0 equal).
5. Elements of columns in N: |x_gpu - x_ref| <= rtol * (|x_ref| + tau_ref).
6. l_{1,1} inner projections: the same rule per column with tau_j; elements
   with ||y| - tau_j| <= rtol * tau_j are near-threshold.
"""
from __future__ import annotations

import numpy as np


def inner_taus(y: np.ndarray, x_ref: np.ndarray) -> np.ndarray:
    """Per-column l1 thresholds recovered from the reference output: for a
    projected column every nonzero output satisfies |x| = |y| - tau_j."""
    d = np.where(x_ref != 0.0, np.abs(y) - np.abs(x_ref), -np.inf)
    return d.max(axis=0)


def check_bilevel(x_gpu, y, ref: dict, q: str, tau_gpu: float | None = None, rtol: float = 1e-5,
                  zero_cols_gpu: int | None = None) -> dict:
    """Assert the parity rule; returns a small report."""
    x_gpu = np.asarray(x_gpu, np.float64)
    y = np.asarray(y, np.float64)
    x_ref = ref["X"]
    tau = ref.get("tau", -1.0)
    v = ref["v"]
    n, m = x_ref.shape
    near = np.zeros(m, bool)
    if tau is not None and tau > 0:
        near = np.abs(v - tau) <= rtol * tau
        if tau_gpu is not None:
            assert abs(tau_gpu - tau) <= rtol * tau, (tau_gpu, tau)
    tol = rtol * np.abs(x_ref)
    if tau is not None and tau > 0:
        tol = tol + np.where(near[None, :], rtol * tau, 0.0)
    if q in ("1", 0):
        taus = inner_taus(y, x_ref)
        has = np.isfinite(taus) & (taus > 0)
        band = has[None, :] & (np.abs(np.abs(y) - taus[None, :]) <= rtol * np.where(has, taus, 0.0)[None, :])
        tol = tol + np.where(band, rtol * np.where(has, taus, 0.0)[None, :], 0.0)
        # columns whose budget itself is near-threshold inherit the outer slack
        tol = tol + np.where(near[None, :], rtol * np.abs(y), 0.0)
    err = np.abs(x_gpu - x_ref)
    bad = err > tol
    assert not bad.any(), (f"{int(bad.sum())} elements out of tolerance; worst at "
                           f"{np.unravel_index(np.argmax(err - tol), err.shape)}: gpu="
                           f"{x_gpu.reshape(-1)[np.argmax(err - tol)]!r} ref={x_ref.reshape(-1)[np.argmax(err - tol)]!r}")
    zg = np.all(x_gpu == 0.0, axis=0)
    zr = np.all(x_ref == 0.0, axis=0)
    assert not np.any((zg != zr) & ~near), "zeroed-column sets differ outside the near-threshold band"
    if zero_cols_gpu is not None:
        assert abs(zero_cols_gpu - ref["zero_columns"]) <= int(near.sum()), (zero_cols_gpu, ref["zero_columns"])
    rel = err / np.maximum(np.abs(x_ref), 1e-300)
    return {"max_rel": float(rel[x_ref != 0].max()) if np.any(x_ref != 0) else 0.0,
            "near": int(near.sum()), "zero_columns": int(zr.sum())}
