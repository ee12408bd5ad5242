"""CPU: the C restatement of l2_error / project / eval_solution (oracle/dg_oracle.c) against the
live reference (oracle/_ref) bitwise, and the quadrature-order rule of dgb_l2_quad_order.
SURVEY.md §8(f) rank 4."""
import os

import numpy as np
import pytest

from oracle.oracle import REF_SO, OracleLib, RefLib
from paper_1502_02941_b200 import capi, dgfem, problems

needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built here")


@pytest.fixture(scope="module")
def orc():
    return OracleLib()


def test_l2_quad_order_rule():
    lib = capi.load()
    # max(2k+3, delivered degree of triangle_rule(quad_order or 2k+2) + 1)
    assert lib.dgb_l2_quad_order(1, 0) == 5       # rule 4 -> 5; 2k+3 = 5
    assert lib.dgb_l2_quad_order(2, 0) == 7       # rule(6) delivers 6 -> 7 = 2k+3
    assert lib.dgb_l2_quad_order(2, 5) == 7
    assert lib.dgb_l2_quad_order(3, 7) == 9       # rule(7) delivers 8 -> 9
    assert lib.dgb_l2_quad_order(4, 0) == 11


@needs_ref
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_postprocess_oracle_matches_reference(orc, k):
    lib = RefLib()
    m = dgfem.unit_square_mesh(6, 0.2, 8 + k, True, 9 + k)
    raw = m.raw()
    rmesh = lib.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
    rref = lib.reference(k, 0)
    nl = rref.tables["n_local"]
    coef = 2.0 * problems.uniform01(31 + k, m.n_elements * nl) - 1.0
    exact = problems.function(capi.FN_SIN_SIN, (1.0,))
    sharp = dgfem.ReferenceElement(k, capi.load().dgb_l2_quad_order(k, 0)).tables()
    assert orc.l2_error(m.arrays(), sharp, coef, exact) == lib.l2_error(rmesh, rref, coef, exact)
    f = problems.function(capi.FN_GAUSSIAN, (50.0, 0.5, 0.5))
    np.testing.assert_array_equal(orc.project(m.arrays(), dgfem.ReferenceElement(k).tables(), f),
                                  lib.project(rmesh, rref, f, m.n_elements))
    rng = np.random.default_rng(k)
    el = rng.integers(0, m.n_elements, 200).astype(np.int32)
    xh = rng.random(200) * 0.5
    yh = rng.random(200) * 0.5
    np.testing.assert_array_equal(orc.eval_solution(coef, k, el, xh, yh),
                                  lib.eval_solution(coef, rref, el, xh, yh))


GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "postprocess.npz")


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_postprocess_oracle_matches_golden(orc, k):
    z = np.load(GOLDEN)
    m = dgfem.build_mesh(z["in_nodes"], z["in_elements"], z["in_dirichlet"], z["in_neumann"])
    coef = z[f"k{k}/coef"]
    exact = problems.function(capi.FN_SIN_SIN, (1.0,))
    sharp = dgfem.ReferenceElement(k, capi.load().dgb_l2_quad_order(k, 0)).tables()
    np.testing.assert_array_equal(np.array(orc.l2_error(m.arrays(), sharp, coef, exact)), z[f"k{k}/l2"])
    f = problems.function(capi.FN_GAUSSIAN, (50.0, 0.5, 0.5))
    np.testing.assert_array_equal(orc.project(m.arrays(), dgfem.ReferenceElement(k).tables(), f),
                                  z[f"k{k}/project"])
    np.testing.assert_array_equal(orc.eval_solution(coef, k, z[f"k{k}/el"], z[f"k{k}/xh"], z[f"k{k}/yh"]),
                                  z[f"k{k}/eval"])
