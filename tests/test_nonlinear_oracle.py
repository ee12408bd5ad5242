"""CPU: the restatement of dgfem::assemble_nonlinear (oracle/dg_oracle.c) pinned bitwise against
fixtures produced by the reference itself (tests/golden/make_golden.py -> nonlinear.npz) and,
where oracle/_ref was built, against the live reference; plus the reference tests' properties
(test_nonlinear.cpp) on the restatement.  SURVEY.md §8(f) rank 1."""
import os

import numpy as np
import pytest

from oracle.oracle import OracleLib, RefLib, ReferenceError_, REF_SO
from paper_1502_02941_b200 import capi, dgfem, problems

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "nonlinear.npz")


@pytest.fixture(scope="module")
def orc():
    return OracleLib()


@pytest.fixture(scope="module")
def z():
    return np.load(GOLDEN)


def case_names(zz):
    return sorted({k.split("/")[0] for k in zz.files if k.endswith("/h")})


def rebuild(zz, name):
    mesh = dgfem.build_mesh(zz[f"{name}/in_nodes"], zz[f"{name}/in_elements"],
                            zz[f"{name}/in_dirichlet"], zz[f"{name}/in_neumann"])
    ref = dgfem.ReferenceElement(int(zz[f"{name}/degree"]), int(zz[f"{name}/quad_order"]))
    return mesh, ref, zz[f"{name}/coef"], int(zz[f"{name}/kind"])


def blocks_to_csr(hj):
    """Block-diagonal HJ [E, nl, nl] -> the reference's CSR (sorted columns)."""
    E, nl, _ = hj.shape
    n = E * nl
    ro = np.arange(0, n * nl + 1, nl, dtype=np.int32)
    cols = (np.repeat(np.arange(E), nl * nl) * nl + np.tile(np.arange(nl), E * nl)).astype(np.int32)
    return ro, cols, hj.reshape(-1)


def test_golden_cases_present(z):
    names = case_names(z)
    assert len(names) == 2 * 4 * 2 * 4  # meshes x degrees x quad orders x reactions
    assert int(z["length_error/status"]) == capi.STATUS_NAMES.index("DimensionMismatch")


@pytest.mark.parametrize("name", case_names(np.load(GOLDEN)))
def test_oracle_matches_reference_bitwise(orc, z, name):
    mesh, ref, coef, kind = rebuild(z, name)
    # the host builders reproduce the reference's mesh and tables exactly (test_host.py)
    h, hj = orc.assemble_nonlinear(mesh.arrays(), ref.tables(), coef, kind, threads=1)
    np.testing.assert_array_equal(h.reshape(-1), z[f"{name}/h"])
    ro, cols, vals = blocks_to_csr(hj)
    np.testing.assert_array_equal(ro, z[f"{name}/row_offsets"])
    np.testing.assert_array_equal(cols, z[f"{name}/cols"])
    np.testing.assert_array_equal(vals, z[f"{name}/vals"])


def test_oracle_length_check(orc):
    mesh = dgfem.unit_square_mesh(4)
    ref = dgfem.ReferenceElement(1)
    with pytest.raises(ReferenceError_) as e:
        orc.assemble_nonlinear(mesh.arrays(), ref.tables(), np.zeros(7), capi.REACTION_SQUARE)
    assert e.value.code == "DimensionMismatch"


def test_oracle_row_subset_and_threads(orc):
    mesh = dgfem.unit_square_mesh(8, 0.2, 5, True, 6)
    ref = dgfem.ReferenceElement(3)
    coef = 2.0 * problems.uniform01(99, mesh.n_elements * ref.n_local) - 1.0
    h, hj = orc.assemble_nonlinear(mesh.arrays(), ref.tables(), coef, capi.REACTION_CUBIC, threads=1)
    h4, hj4 = orc.assemble_nonlinear(mesh.arrays(), ref.tables(), coef, capi.REACTION_CUBIC, threads=4)
    np.testing.assert_array_equal(h, h4)
    np.testing.assert_array_equal(hj, hj4)
    rows = np.array([5, 0, 77, mesh.n_elements - 1], np.int32)
    hs, hjs = orc.assemble_nonlinear(mesh.arrays(), ref.tables(), coef, capi.REACTION_CUBIC, rows=rows)
    np.testing.assert_array_equal(hs, h[rows])
    np.testing.assert_array_equal(hjs, hj[rows])


def test_linear_reaction_is_the_mass_matrix(orc):
    """test_nonlinear.cpp:67-92: r(u) = u gives HJ = the alpha = 1 mass matrix and H = HJ coef."""
    mesh = dgfem.unit_square_mesh(4, 0.1, 1, False, 0)
    ref = dgfem.ReferenceElement(2)
    nl = ref.n_local
    coef = 2.0 * problems.uniform01(101, mesh.n_elements * nl) - 1.0
    h, hj = orc.assemble_nonlinear(mesh.arrays(), ref.tables(), coef, capi.REACTION_LINEAR)
    # mass blocks of the linear assembly: K with eps = 0, b = 0, alpha = 1, no faces -> R
    hc = np.einsum("eij,ej->ei", hj, coef.reshape(-1, nl))
    assert np.abs(hc - h).max() <= 1e-12
    assert np.abs(hj - np.transpose(hj, (0, 2, 1))).max() == 0.0


def test_zero_coefficients_give_zero(orc):
    mesh = dgfem.unit_square_mesh(4)
    ref = dgfem.ReferenceElement(2)
    h, hj = orc.assemble_nonlinear(mesh.arrays(), ref.tables(), np.zeros(mesh.n_elements * 6),
                                   capi.REACTION_SQUARE)
    assert not h.any() and not hj.any()


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built here")
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_oracle_matches_live_reference(orc, k):
    lib = RefLib()
    m = dgfem.unit_square_mesh(7, 0.2, 40 + k, True, 50 + k, 2 | 8)
    raw = m.raw()
    rmesh = lib.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
    rref = lib.reference(k, 0)
    ref = dgfem.ReferenceElement(k)
    coef = 2.0 * problems.uniform01(7 + k, m.n_elements * ref.n_local) - 1.0
    for kind in (capi.REACTION_SQUARE, capi.REACTION_CUBIC):
        h_ref, (ro, cols, vals), _ = lib.assemble_nonlinear(rmesh, rref, coef, kind)
        h, hj = orc.assemble_nonlinear(m.arrays(), ref.tables(), coef, kind)
        np.testing.assert_array_equal(h.reshape(-1), h_ref)
        np.testing.assert_array_equal(blocks_to_csr(hj)[2], vals)
