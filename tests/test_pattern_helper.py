"""The mesh-derived pattern the full-size GPU tests compare against (helpers.expected_pattern)
equals the oracle's pattern (pinned to the reference's stiffness() CSR)."""
import numpy as np
import pytest

from helpers import expected_pattern
from oracle.oracle import OracleLib
from paper_1502_02941_b200 import capi, dgfem, problems


@pytest.mark.parametrize("n,jitter,permute,neumann", [(5, 0.0, False, 0), (9, 0.2, True, 2 | 8),
                                                      (7, 0.1, True, 15)])
def test_expected_pattern_equals_oracle(n, jitter, permute, neumann):
    mesh = dgfem.unit_square_mesh(n, jitter, 3, permute, 4, neumann)
    ref = dgfem.ReferenceElement(1, 3)
    spec = problems.config_problem(1)
    params = dgfem.set_parameters(capi.SIPG, 1, capi.INFLOW_DROP)
    rp, col, _, _ = OracleLib().assemble(mesh.arrays(), ref.tables(), spec.c, params)
    erp, ecol = expected_pattern(mesh.arrays())
    assert np.array_equal(rp, erp)
    assert np.array_equal(col, ecol)
