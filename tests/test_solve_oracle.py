"""CPU: the solve-layer restatement (oracle/newton.py; SuperLU standing in for Eigen's
SparseLU, which is not in this image) against the reference's own tests of that layer
(test_nonlinear.cpp:164-240): one Newton step for a vanishing reaction, convergence within
budget on the boundary-layer problem, quadratic convergence on a smooth cubic problem.
SURVEY.md §8(f) rank 2."""
import numpy as np
import pytest

from oracle import newton as onewton
from oracle.oracle import OracleLib, bsr_to_csr
from paper_1502_02941_b200 import capi, dgfem, problems


@pytest.fixture(scope="module")
def orc():
    return OracleLib()


def system(orc, name, degree, n=4, method=capi.SIPG):
    spec = problems.registry_get(name)
    mesh = dgfem.unit_square_mesh(n, 0.0, 0, False, 0, spec.neumann_sides)
    tables = dgfem.ReferenceElement(degree).tables()
    p = dgfem.set_parameters(method, degree)
    rp, col, val, rhs = orc.assemble(mesh.arrays(), tables, spec.c, p)
    return mesh, tables, bsr_to_csr(rp, col, val), rhs.reshape(-1)


def test_direct_solve_meets_the_contract(orc):
    _, _, (ro, ci, va), F = system(orc, "smooth-sine", 2)
    x, info = onewton.direct_solve(ro, ci, va, F)
    assert info["defect_norm2"] <= info["bound"]
    with pytest.raises(onewton.SingularMatrixError):
        onewton.direct_solve(ro, ci, np.zeros_like(va), F)


def test_newton_linear_problem_one_step(orc):
    """test_nonlinear.cpp:164-182: zero reaction -> exactly one step, equal to the direct solve."""
    mesh, tables, K, F = system(orc, "smooth-sine", 1)
    coef, rep = onewton.newton_solve(K, F, mesh.arrays(), tables, capi.REACTION_ZERO, orc)
    assert rep["iterations"] == 1 and rep["converged"] and len(rep["residual_history"]) == 1
    assert rep["final_residual"] <= 1e-10
    x, _ = onewton.direct_solve(*K, F)
    assert np.all(np.abs(coef - x) <= 1e-12 * np.maximum(1.0, np.abs(x)))


def test_newton_layer_problem_within_budget(orc):
    """test_nonlinear.cpp:184-199 (with the linear variant's data and r(u) = u^2)."""
    mesh, tables, K, F = system(orc, "paper-boundary-layer-linear", 1, n=8)
    coef, rep = onewton.newton_solve(K, F, mesh.arrays(), tables, capi.REACTION_SQUARE, orc)
    assert rep["converged"] and rep["iterations"] <= 50 and rep["final_residual"] <= 1e-10
    assert np.all(np.isfinite(coef))


def test_newton_cubic_converges_quadratically(orc):
    """test_nonlinear.cpp:201-240: the last steps shrink the residual quadratically."""
    mesh, tables, K, F = system(orc, "smooth-sine", 2, n=6)
    _, rep = onewton.newton_solve(K, 10.0 * F, mesh.arrays(), tables, capi.REACTION_CUBIC, orc)
    h = rep["residual_history"]
    assert rep["converged"] and len(h) >= 3
    # quadratic: r_{k+1} <= C r_k^2 once in the basin
    assert h[-2] <= 1e-3 * max(h[-3], 1e-300) ** 1.0 or h[-2] <= 10 * h[-3] ** 2
