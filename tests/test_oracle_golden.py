"""CPU: the plain-C restatement oracle pinned against fixtures produced by the reference itself
(tests/golden/make_golden.py), and -- where oracle/_ref was built -- against the live reference."""
import os

import numpy as np
import pytest

from oracle.oracle import OracleLib, RefLib, ReferenceError_, bsr_to_csr
from paper_1502_02941_b200 import capi, dgfem, problems
from paper_1502_02941_b200.capi import Params

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def orc():
    return OracleLib()


@pytest.fixture(scope="module")
def systems():
    return np.load(os.path.join(GOLDEN, "systems.npz"))


def case_names(z):
    return sorted({k.split("/")[0] for k in z.files if k.endswith("/row_offsets")})


def rebuild(z, name):
    """Mesh (via the host builder), tables, problem and params of a golden system case."""
    mesh = dgfem.build_mesh(z[f"{name}/in_nodes"], z[f"{name}/in_elements"],
                            z[f"{name}/in_dirichlet"], z[f"{name}/in_neumann"])
    k, qo = int(z[f"{name}/degree"]), int(z[f"{name}/quad_order"])
    tables = dgfem.ReferenceElement(k, qo).tables()
    pv = z[f"{name}/params"]
    p = Params()
    p.method, p.degree, p.kappa = int(pv[0]), int(pv[1]), pv[2]
    p.sigma_interior, p.sigma_boundary, p.neumann_inflow = pv[3], pv[4], int(pv[5])
    if name.startswith("config"):
        spec = problems.config_problem(int(name[6]), mesh.n_elements)
    elif name.startswith("two_element"):
        spec = problems.registry_get("poly-exact")
        spec.c.advection = problems.vec_constant(2.0, 1.0)
    else:
        spec = problems.registry_get(name.rsplit("_k", 1)[0])
    for field in ("diffusion", "linear_reaction"):
        key = f"{name}/per_element_{field}"
        if key in z.files:
            np.testing.assert_array_equal(spec.per_element[field], z[key])
    return mesh, tables, spec, p


def test_golden_cases_present(systems):
    names = case_names(systems)
    for idx in (1, 2, 3, 4, 5):
        assert any(n.startswith(f"config{idx}_") for n in names)
    assert len(names) >= 14


@pytest.mark.parametrize("name", case_names(np.load(os.path.join(GOLDEN, "systems.npz"))))
def test_oracle_matches_reference_bitwise(orc, systems, name):
    """K = stiffness() pattern and values, and F, bitwise equal to the reference's output."""
    mesh, tables, spec, p = rebuild(systems, name)
    rp, col, val, rhs = orc.assemble(mesh.arrays(), tables, spec.c, p, threads=2)
    crp, ccol, cval = bsr_to_csr(rp, col, val)
    np.testing.assert_array_equal(crp, systems[f"{name}/row_offsets"])
    np.testing.assert_array_equal(ccol, systems[f"{name}/cols"])
    np.testing.assert_array_equal(cval, systems[f"{name}/vals"])
    np.testing.assert_array_equal(rhs.reshape(-1), systems[f"{name}/F"])


def test_oracle_row_subsets_equal_full(orc, systems):
    """Any subset of block rows equals the same rows of the full assembly (bitwise)."""
    name = "config3_sipg"
    mesh, tables, spec, p = rebuild(systems, name)
    full = orc.assemble(mesh.arrays(), tables, spec.c, p)
    rows = np.array([0, 5, 17, 18, 40, mesh.n_elements - 1], np.int32)
    sub = orc.assemble(mesh.arrays(), tables, spec.c, p, rows=rows)
    for r_i, r in enumerate(rows):
        b0, b1 = full[0][r], full[0][r + 1]
        s0, s1 = sub[0][r_i], sub[0][r_i + 1]
        np.testing.assert_array_equal(full[1][b0:b1], sub[1][s0:s1])
        np.testing.assert_array_equal(full[2][b0:b1], sub[2][s0:s1])
        np.testing.assert_array_equal(full[3][r], sub[3][r_i])


def test_oracle_thread_count_independent(orc, systems):
    """test_parallel_consistency.cpp:59-105: bitwise identical for any thread count."""
    mesh, tables, spec, p = rebuild(systems, "config2_nipg")
    a = orc.assemble(mesh.arrays(), tables, spec.c, p, threads=1)
    for t in (2, 3, 7):
        b = orc.assemble(mesh.arrays(), tables, spec.c, p, threads=t)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


def test_oracle_inflow_on_neumann_detail(orc, systems):
    """test_assembly.cpp:371-381 + test_parallel_consistency.cpp:152-182: InflowOnNeumann with
    the reference's (lowest) offending edge."""
    z = systems
    mesh = dgfem.build_mesh(z["inflow_on_neumann/in_nodes"], z["inflow_on_neumann/in_elements"],
                            z["inflow_on_neumann/in_dirichlet"], z["inflow_on_neumann/in_neumann"])
    tables = dgfem.ReferenceElement(1).tables()
    with pytest.raises(ReferenceError_) as err:
        orc.assemble(mesh.arrays(), tables, problems.registry_get("smooth-sine").c,
                     dgfem.set_parameters(capi.SIPG, 1))
    assert err.value.code == "InflowOnNeumann"
    assert err.value.detail == int(z["inflow_on_neumann/detail"])


def test_oracle_spmv_matches_csr_matvec(orc, systems):
    """matvec (sparse.cpp:116-129) over the expanded CSR equals dgo_spmv bitwise."""
    mesh, tables, spec, p = rebuild(systems, "config4_sipg")
    rp, col, val, _ = orc.assemble(mesh.arrays(), tables, spec.c, p)
    x = np.random.default_rng(3).uniform(-1, 1, mesh.n_elements * tables["n_local"])
    y = orc.spmv(rp, col, val, x)
    crp, ccol, cval = bsr_to_csr(rp, col, val)
    y2 = np.array([sum(cval[k] * x[ccol[k]] for k in range(crp[r], crp[r + 1]))
                   for r in range(crp.shape[0] - 1)])
    np.testing.assert_array_equal(y, y2)


# --------------------------------------------------------------------------- properties
def _sym_spec():
    """Pure diffusion (b = 0, alpha = 0): K = D."""
    spec = problems.registry_get("smooth-sine")
    spec.c.advection = problems.vec_constant(0.0, 0.0)
    spec.c.linear_reaction = problems.constant(0.0)
    return spec


def test_sipg_diffusion_bitwise_symmetric(orc):
    """test_assembly.cpp:263-279: SIPG D is bitwise symmetric (reference property, kept by the
    restatement)."""
    mesh = dgfem.unit_square_mesh(5, 0.2, 1, True, 2, 0)
    for k in (1, 2, 3):
        tables = dgfem.ReferenceElement(k).tables()
        rp, col, val, _ = orc.assemble(mesh.arrays(), tables, _sym_spec().c,
                                       dgfem.set_parameters(capi.SIPG, k))
        crp, ccol, cval = bsr_to_csr(rp, col, val)
        n = crp.shape[0] - 1
        import scipy.sparse as sp
        K = sp.csr_matrix((cval, ccol, crp), shape=(n, n))
        assert abs(K - K.T).max() == 0.0


def test_nipg_iipg_not_symmetric(orc):
    """test_assembly.cpp:281-291."""
    import scipy.sparse as sp
    mesh = dgfem.unit_square_mesh(2)
    tables = dgfem.ReferenceElement(1).tables()
    for m in (capi.NIPG, capi.IIPG):
        rp, col, val, _ = orc.assemble(mesh.arrays(), tables, _sym_spec().c,
                                       dgfem.set_parameters(m, 1))
        crp, ccol, cval = bsr_to_csr(rp, col, val)
        K = sp.csr_matrix((cval, ccol, crp))
        assert abs(K - K.T).max() > 1e-6


def test_mass_blocks_are_scaled_identities(orc):
    """test_assembly.cpp:383-406 / acceptance #6: R blocks = det * I (diffusion and transport
    switched off)."""
    mesh = dgfem.unit_square_mesh(3, 0.2, 9, False, 0, 0)
    for k in (1, 2):
        spec = problems.make_problem("mass", 0.0, problems.vec_constant(0.0, 0.0), 1.0,
                                     problems.constant(0.0), problems.constant(0.0))
        p = dgfem.set_parameters(capi.SIPG, k)
        p.sigma_interior = p.sigma_boundary = 0.0
        tables = dgfem.ReferenceElement(k).tables()
        rp, col, val, _ = orc.assemble(mesh.arrays(), tables, spec.c, p)
        nodes, el = mesh.nodes, mesh.elements
        for e in range(mesh.n_elements):
            p0, p1, p2 = nodes[el[e]]
            det = (p1[0] - p0[0]) * (p2[1] - p0[1]) - (p2[0] - p0[0]) * (p1[1] - p0[1])
            for b in range(rp[e], rp[e + 1]):
                expect = det * np.eye(tables["n_local"]) if col[b] == e else 0.0
                assert np.abs(val[b] - expect).max() <= 1e-12


def test_load_is_bitwise_linear_in_source(orc):
    """test_assembly.cpp:447-471: scaling f by 4 scales F bitwise (zero boundary data)."""
    mesh = dgfem.unit_square_mesh(4, 0.1, 2, False, 0, 0)
    tables = dgfem.ReferenceElement(2).tables()
    spec = problems.make_problem("lin", 1.0, problems.vec_constant(1.0, 2.0), 1.0,
                                 problems.function(capi.FN_SIN_SIN, (1.0,)), problems.constant(0.0))
    p = dgfem.set_parameters(capi.SIPG, 2)
    F1 = orc.assemble(mesh.arrays(), tables, spec.c, p)[3]
    spec.c.source.p[0] = 4.0
    F4 = orc.assemble(mesh.arrays(), tables, spec.c, p)[3]
    np.testing.assert_array_equal(F4, 4.0 * F1)


# --------------------------------------------------------------------------- live reference
ref_required = pytest.mark.skipif(not os.path.exists(os.path.join(
    os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref", "libdgref.so")),
    reason="oracle/_ref not built (no /root/reference here)")


@ref_required
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_oracle_matches_live_reference_random_meshes(orc, k):
    """Fresh seeded meshes / coefficients, every method: restatement == reference bitwise."""
    ref = RefLib()
    rng = np.random.default_rng(k)
    for trial in range(2):
        n = int(rng.integers(2, 5))
        sides = int(rng.integers(0, 16))
        m = dgfem.unit_square_mesh(n, 0.2, int(rng.integers(1 << 30)), bool(trial), 5, sides)
        raw = m.raw()
        rm = ref.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
        spec = problems.registry_get("smooth-sine")
        spec.c.advection = problems.vec_affine(0.3, -0.2, 0.5, -1.0, 1.0, 0.25)
        spec.set_per_element("diffusion", rng.uniform(0.1, 2.0, m.n_elements))
        spec.set_per_element("linear_reaction", rng.uniform(0.0, 2.0, m.n_elements))
        rr = ref.reference(k, 2 * k + 1)
        for meth in (capi.SIPG, capi.NIPG, capi.IIPG):
            p = dgfem.set_parameters(meth, k, capi.INFLOW_DROP)
            s = ref.assemble(rm, rr, spec.c, p, threads=2, clip_sides=sides)
            rp, col, val, rhs = orc.assemble(m.arrays(), rr.tables, spec.c, p)
            crp, ccol, cval = bsr_to_csr(rp, col, val)
            grp, gcol, gval = s.csr(0)
            np.testing.assert_array_equal(crp, grp)
            np.testing.assert_array_equal(ccol, gcol)
            np.testing.assert_array_equal(cval, gval)
            np.testing.assert_array_equal(rhs.reshape(-1), s.rhs())
