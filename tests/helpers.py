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


def expected_pattern(mesh: dict):
    """The reference's K pattern (SURVEY.md §8 "K pattern": the diagonal block plus both
    off-diagonal blocks of every interior edge, block columns sorted ascending, as
    `stiffness()`'s CSR has them, sparse.cpp:46-51) computed in numpy from the mesh arrays
    alone: (row_ptr [E+1], col [E+2I]).  Size-independent, so it checks the GPU pattern of a
    full-size config bit for bit."""
    ee = mesh["element_edges"].astype(np.int64)                  # [E, 3]
    lr = mesh["edge_elements"][ee]                               # [E, 3, 2]
    E = ee.shape[0]
    me = np.arange(E, dtype=np.int64)[:, None]
    nb = np.where(lr[..., 0] == me, lr[..., 1], lr[..., 0]).astype(np.int64)
    big = np.iinfo(np.int64).max
    nb = np.where(nb < 0, big, nb)
    cols = np.sort(np.concatenate([me, nb], axis=1), axis=1)     # [E, 4]
    keep = cols != big
    row_ptr = np.zeros(E + 1, np.int32)
    row_ptr[1:] = np.cumsum(keep.sum(axis=1))
    return row_ptr, cols[keep].astype(np.int32)


def sample_rows(n_rows: int, seed: int, n_sample: int = 4000, edge: int = 64) -> np.ndarray:
    """A seeded sample of block rows plus the first and last `edge` rows (sorted, unique)."""
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([
        rng.choice(n_rows, size=min(n_rows, n_sample), replace=False),
        np.arange(min(edge, n_rows)), np.arange(max(0, n_rows - edge), n_rows)]))


def gather_rows_device(out, rows):
    """Block rows `rows` of a device BsrSystem, gathered on the device and copied back in the
    oracle's subset layout (avoids copying a multi-GB full matrix to the host)."""
    import torch
    rows = np.asarray(rows)
    rp = out.row_ptr.cpu().numpy()
    counts = rp[rows + 1] - rp[rows]
    out_rp = np.zeros(rows.size + 1, np.int32)
    out_rp[1:] = np.cumsum(counts)
    idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
    it = torch.from_numpy(idx).to(out.val.device)
    ir = torch.from_numpy(rows.astype(np.int64)).to(out.val.device)
    return (out_rp, out.col[it].cpu().numpy(), out.val[it].cpu().numpy(),
            out.rhs[ir].cpu().numpy())
