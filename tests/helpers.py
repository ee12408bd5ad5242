"""Shared checks: the comparator of SURVEY.md §8(c)."""
from __future__ import annotations

import numpy as np

TOL = 1e-12  # north_star: max relative error 1e-12, per-row scaled


def row_scale(val: np.ndarray, row_ptr: np.ndarray) -> np.ndarray:
    """max_j |K_ij| per scalar row i, for a BSR with val [nb, nl, nl] -> [n_rows, nl]."""
    nl = val.shape[1]
    blockmax = np.abs(val).max(axis=2)                       # [nb, nl]
    n = row_ptr.shape[0] - 1
    out = np.zeros((n, nl))
    counts = np.diff(row_ptr)
    owner = np.repeat(np.arange(n), counts)
    np.maximum.at(out, owner, blockmax)
    return out


def compare_system(gpu, ref, tol: float = TOL) -> dict:
    """gpu / ref = (row_ptr, col, val[nb,nl,nl], rhs[n,nl]) for the same block rows.
    Pattern must be bit-exact; K entries within tol * row max; F within tol * block max."""
    g_rp, g_col, g_val, g_rhs = gpu
    r_rp, r_col, r_val, r_rhs = ref
    assert np.array_equal(g_rp, r_rp), "row_ptr differs"
    assert np.array_equal(g_col, r_col), "block column indices differ"
    scale = row_scale(r_val, r_rp)                           # [n, nl]
    counts = np.diff(r_rp)
    owner = np.repeat(np.arange(r_rp.shape[0] - 1), counts)
    s = np.maximum(scale[owner][:, :, None], 1e-300)
    kerr = float((np.abs(g_val - r_val) / s).max()) if r_val.size else 0.0
    fscale = np.maximum(np.abs(r_rhs).max(axis=1, keepdims=True), 1e-300)
    ferr = float((np.abs(g_rhs - r_rhs) / fscale).max()) if r_rhs.size else 0.0
    assert kerr <= tol, f"K max row-scaled error {kerr:.3e} > {tol}"
    assert ferr <= tol, f"F max block-scaled error {ferr:.3e} > {tol}"
    return {"K": kerr, "F": ferr}


def gather_rows(rp, col, val, rhs, rows):
    """Extract block rows `rows` from a full BSR (numpy) in the oracle's subset layout."""
    rows = np.asarray(rows)
    counts = rp[rows + 1] - rp[rows]
    out_rp = np.zeros(rows.size + 1, np.int32)
    out_rp[1:] = np.cumsum(counts)
    idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows]) if rows.size else np.zeros(0, int)
    return out_rp, col[idx], val[idx], rhs[rows]
