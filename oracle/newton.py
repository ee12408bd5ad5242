"""TEST INFRASTRUCTURE -- never imported by the product.

numpy restatement of the reference's solve layer for the parity tests of SURVEY.md §8(f)
rank 2:

* `direct_solve` (sparse.cpp:154-217): the reference factorises with Eigen 3 (>= 3.3,
  CMakeLists.txt:12) SparseLU, which is neither vendored in /root/reference nor installed
  here.  SciPy's SuperLU (scipy.sparse.linalg.splu, sparse LU with partial pivoting and a
  fill-reducing column order -- the same published algorithm family) stands in for it.  The
  acceptance test (defect <= 1e-10 (||A||_F ||x|| + ||b||)) is restated exactly.
* `newton_solve` (nonlinear.cpp:109-176): restated line by line on top of it, with
  H / HJ from the C restatement of assemble_nonlinear (dg_oracle.c, pinned bitwise to the
  reference by tests/test_nonlinear_oracle.py).

Parity is anchored on the reference's own tests of this layer (test_nonlinear.cpp:177-240,
test_sparse.cpp): a vanishing reaction converges in exactly one Newton step to the direct
solution, the boundary-layer problem converges within budget, the cubic problem converges
quadratically.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class SolveAccuracyError(RuntimeError):
    pass


class SingularMatrixError(RuntimeError):
    pass


def direct_solve(row_offsets, cols, vals, rhs):
    """x with the reference's defect report; raises SolveAccuracyError like sparse.cpp:212."""
    n = row_offsets.shape[0] - 1
    a = sp.csr_matrix((vals, cols, row_offsets), shape=(n, n))
    try:
        x = spla.splu(a.tocsc()).solve(np.asarray(rhs, dtype=np.float64))
    except RuntimeError as e:  # "Factor is exactly singular" -> the reference's SingularMatrix
        raise SingularMatrixError(str(e)) from e
    d = a @ x - rhs
    defect2 = float(np.sqrt(np.sum(d * d)))
    bound = 1e-10 * (float(np.sqrt(np.sum(vals * vals))) * float(np.sqrt(np.sum(x * x)))
                     + float(np.sqrt(np.sum(rhs * rhs))))
    info = {"defect_norm2": defect2, "defect_norm_inf": float(np.abs(d).max()) if n else 0.0,
            "bound": bound}
    if defect2 > bound:
        raise SolveAccuracyError("direct solve defect exceeds accuracy bound")
    return x, info


def bsr_csr(row_ptr, col, val):
    from oracle.oracle import bsr_to_csr
    return bsr_to_csr(row_ptr, col, val)


def newton_solve(K_csr, F, mesh_arrays, tables, kind, orc, max_iterations=50,
                 residual_tolerance=1e-10, step_tolerance=1e-12, initial_guess=None):
    """nonlinear.cpp:109-176 with H/HJ from the restatement `orc` (OracleLib)."""
    ro, ci, va = K_csr
    n = ro.shape[0] - 1
    nl = tables["n_local"]
    K = sp.csr_matrix((va, ci, ro), shape=(n, n))
    coef = np.zeros(n) if initial_guess is None else np.array(initial_guess, dtype=np.float64)

    def evaluate():
        h, hj = orc.assemble_nonlinear(mesh_arrays, tables, coef, kind)
        res = K @ coef + h.reshape(-1) - F
        E = hj.shape[0]
        blocks = (sp.block_diag([sp.csr_matrix(hj[e]) for e in range(E)], format="csr")
                  if E else sp.csr_matrix((0, 0)))
        return res, blocks

    report = {"iterations": 0, "converged": False, "final_residual": 0.0, "residual_history": []}
    residual, hj = evaluate()
    for it in range(max_iterations):
        J = (K + hj).tocsr()
        J.sort_indices()
        step, _ = direct_solve(J.indptr, J.indices, J.data, -residual)
        coef += step
        report["iterations"] = it + 1
        res_new, hj = evaluate()
        res_norm = float(np.sqrt(np.sum(res_new * res_new)))
        report["residual_history"].append(res_norm)
        report["final_residual"] = res_norm
        if res_norm <= residual_tolerance or float(np.sqrt(np.sum(step * step))) <= step_tolerance:
            report["converged"] = True
            break
        residual = res_new
    return coef, report
