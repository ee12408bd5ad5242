"""oracle/meshgen.py (the numpy generator the reference arm feeds to the reference's
build_mesh) is bit-identical to the library's dgb_mesh_rectangle."""
import numpy as np
import pytest

from oracle import meshgen
from paper_1502_02941_b200 import dgfem, problems


@pytest.mark.parametrize("n,jitter,permute,neumann", [(4, 0.0, False, 0), (16, 0.2, False, 2 | 8),
                                                      (13, 0.0, True, 0), (11, 0.3, True, 15)])
def test_meshgen_matches_library(n, jitter, permute, neumann):
    raw = meshgen.unit_square_raw(n, jitter, problems.SEED_JITTER, permute, problems.SEED_PERMUTE,
                                  neumann)
    lib = dgfem.unit_square_mesh(n, jitter, problems.SEED_JITTER, permute, problems.SEED_PERMUTE,
                                 neumann).raw()
    for k in ("nodes", "elements", "dirichlet", "neumann"):
        assert raw[k].shape == lib[k].shape, k
        assert np.array_equal(raw[k], lib[k]), k


def test_meshgen_rectangle_matches_library():
    raw = meshgen.rectangle_raw(12, 5, 3.0, 1.0, 0.1, 9, True, 10, 4)
    lib = dgfem.rectangle_mesh(12, 5, 3.0, 1.0, 0.1, 9, True, 10, 4).raw()
    for k in ("nodes", "elements", "dirichlet", "neumann"):
        assert np.array_equal(raw[k], lib[k]), k
