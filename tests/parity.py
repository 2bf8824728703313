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


def _l1_fiber_taus(v: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Per-fiber l1 thresholds (fibers along axis 0) recovered from norms v and
    projected budgets u: every positive u equals v - tau."""
    d = np.where(u > 0.0, v - u, -np.inf)
    return d.max(axis=0) if d.ndim > 1 else np.asarray(d.max())


def _near_slack(v: np.ndarray, u: np.ndarray, rtol: float) -> np.ndarray:
    """tau_f where an entry's norm is within rtol * tau_f of its fiber's l1
    threshold (its budget may be 0 or up to rtol * tau_f), else 0."""
    tau = _l1_fiber_taus(v, u)
    has = np.isfinite(tau) & (tau > 0)
    tau = np.where(has, tau, 0.0)
    return np.where(has & (np.abs(v - tau) <= rtol * tau), tau, 0.0) * np.ones_like(v)


def check_multilevel(x_gpu, t, levels, x_ref, chain_ref, chain_gpu=None, rtol: float = 1e-5) -> dict:
    """§8(c) rule applied per level of a multi-level projection.

    levels are innermost first (codes 0 = l1, 1 = l2, 2 = inf); chain_ref /
    chain_gpu are budget chains deepest first (U_{r-1}, ..., U_1).  Each budget
    U_k may differ by rtol * (|U_k| + S_k); S_k is the near-threshold slack: an
    entry whose norm lies within rtol * tau of its fiber's l1 threshold tau
    carries tau, and a fiber inherits its parent's slack (the l1 / l2 / inf
    projections move a child budget by at most the move of the radius).
    Elements: rtol * (|x_ref| + S_1), plus the l1 inner band rule of
    check_bilevel when the innermost level is l1."""
    x_gpu = np.asarray(x_gpu, np.float64)
    t = np.asarray(t, np.float64)
    r = len(levels)
    assert r >= 2
    # norm chain V_1 .. V_{r-1} (aggregates over the leading axis)
    V = [None]
    cur = np.abs(t)
    for k in range(r - 1):
        q = levels[k]
        cur = cur.sum(0) if q == 0 else (np.sqrt((cur * cur).sum(0)) if q == 1 else cur.max(0))
        V.append(cur)
    U = [None] * r
    for k, c in zip(range(r - 1, 0, -1), chain_ref):
        U[k] = np.asarray(c, np.float64).reshape(V[k].shape)
    S = [None] * r
    S[r - 1] = _near_slack(V[r - 1], U[r - 1], rtol) if levels[r - 1] == 0 else np.zeros_like(V[r - 1])
    for k in range(r - 2, 0, -1):
        inh = np.broadcast_to(S[k + 1], V[k].shape)
        S[k] = inh + (_near_slack(V[k], U[k], rtol) if levels[k] == 0 else 0.0)
    if chain_gpu is not None:
        for k, c in zip(range(r - 1, 0, -1), chain_gpu):
            ug = np.asarray(c, np.float64).reshape(V[k].shape)
            bad = np.abs(ug - U[k]) > rtol * (np.abs(U[k]) + S[k])
            assert not bad.any(), f"level {k}: {int(bad.sum())} budgets out of tolerance"
    tol = rtol * (np.abs(x_ref) + np.broadcast_to(S[1], t.shape))
    if levels[0] == 0:
        d0 = t.shape[0]
        y2, x2 = t.reshape(d0, -1), np.asarray(x_ref, np.float64).reshape(d0, -1)
        taus = inner_taus(y2, x2)
        has = np.isfinite(taus) & (taus > 0)
        tt = np.where(has, taus, 0.0)[None, :]
        band = has[None, :] & (np.abs(np.abs(y2) - tt) <= rtol * tt)
        tol = tol + np.where(band, rtol * tt, 0.0).reshape(t.shape)
    err = np.abs(x_gpu - x_ref)
    bad = err > tol
    assert not bad.any(), (f"{int(bad.sum())} elements out of tolerance; worst gpu="
                           f"{x_gpu.reshape(-1)[np.argmax(err - tol)]!r} ref={x_ref.reshape(-1)[np.argmax(err - tol)]!r}")
    rel = err / np.maximum(np.abs(x_ref), 1e-300)
    return {"max_rel": float(rel[x_ref != 0].max()) if np.any(x_ref != 0) else 0.0,
            "near_entries": int(sum(int((s > 0).sum()) for s in S[1:]))}
