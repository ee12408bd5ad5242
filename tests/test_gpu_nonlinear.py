"""GPU: dgb_assemble_nonlinear (nonlinear.cpp:11-107) against the
reference's golden fixtures and the C restatement.  H uses the reference's operations in the
reference's order, so it must be BITWISE equal; HJ goes through the FP64 tensor cores and must
be within 1e-12 of the per-row max (the north_star tolerance), bitwise symmetric per block."""
import numpy as np
import pytest

from oracle.oracle import OracleLib
from paper_1502_02941_b200 import capi, dgfem, problems
from test_nonlinear_oracle import GOLDEN, blocks_to_csr, case_names, rebuild

pytestmark = pytest.mark.gpu
TOL = 1e-12


def hj_error(g, r):
    """max |g - r| / max_j |r_ij| over rows of the blocks [E, nl, nl]."""
    s = np.maximum(np.abs(r).max(axis=2, keepdims=True), 1e-300)
    return float((np.abs(g - r) / s).max()) if r.size else 0.0


def device_nonlinear(mesh, ref, coef, kind):
    import torch
    plan = dgfem.Plan(ref.view)
    dm = dgfem.DeviceMesh(mesh)
    h, hj = plan.assemble_nonlinear(dm, torch.from_numpy(np.ascontiguousarray(coef)).cuda(), kind)
    torch.cuda.synchronize()
    return (h.cpu().numpy(), hj.row_ptr.cpu().numpy(), hj.col.cpu().numpy(), hj.val.cpu().numpy())


@pytest.mark.parametrize("name", case_names(np.load(GOLDEN)))
def test_matches_reference_golden(name):
    z = np.load(GOLDEN)
    mesh, ref, coef, kind = rebuild(z, name)
    h, rp, col, val = device_nonlinear(mesh, ref, coef, kind)
    E = mesh.n_elements
    np.testing.assert_array_equal(rp, np.arange(E + 1))
    np.testing.assert_array_equal(col, np.arange(E))
    np.testing.assert_array_equal(h.reshape(-1), z[f"{name}/h"])          # bitwise
    ro, cols, _ = blocks_to_csr(val)
    np.testing.assert_array_equal(ro, z[f"{name}/row_offsets"])
    np.testing.assert_array_equal(cols, z[f"{name}/cols"])
    nl = ref.n_local
    assert hj_error(val, z[f"{name}/vals"].reshape(E, nl, nl)) <= TOL
    np.testing.assert_array_equal(val, np.transpose(val, (0, 2, 1)))       # symmetric, bitwise


def test_host_entry_equals_device_path():
    mesh = dgfem.unit_square_mesh(16, 0.2, 3, True, 4)
    ref = dgfem.ReferenceElement(2)
    coef = 2.0 * problems.uniform01(5, mesh.n_elements * ref.n_local) - 1.0
    h, rp, col, val = device_nonlinear(mesh, ref, coef, capi.REACTION_CUBIC)
    h2, (rp2, col2, val2) = dgfem.assemble_nonlinear(coef, mesh, ref, capi.REACTION_CUBIC)
    np.testing.assert_array_equal(h.reshape(-1), h2)
    np.testing.assert_array_equal(rp, rp2)
    np.testing.assert_array_equal(col, col2)
    np.testing.assert_array_equal(val, val2)


def test_length_mismatch_raises():
    mesh = dgfem.unit_square_mesh(4)
    ref = dgfem.ReferenceElement(1)
    with pytest.raises(dgfem.Error) as e:
        dgfem.assemble_nonlinear(np.zeros(7), mesh, ref, capi.REACTION_SQUARE)
    assert e.value.code == "DimensionMismatch"


@pytest.mark.parametrize("degree", [1, 2, 3, 4])
def test_full_size_sampled_against_oracle(degree):
    """Config-2-sized mesh (256^2 x 2 triangles): H bitwise and HJ within 1e-12 on 4096
    sampled elements recomputed by the restatement."""
    n = 256 if degree <= 2 else 128
    mesh = dgfem.unit_square_mesh(n, 0.2, 11, True, 12)
    ref = dgfem.ReferenceElement(degree)
    nl = ref.n_local
    coef = 2.0 * problems.uniform01(1234 + degree, mesh.n_elements * nl) - 1.0
    h, rp, col, val = device_nonlinear(mesh, ref, coef, capi.REACTION_SQUARE)
    rows = np.unique(np.random.default_rng(degree).integers(0, mesh.n_elements, 4096)).astype(np.int32)
    ho, hjo = OracleLib().assemble_nonlinear(mesh.arrays(), ref.tables(), coef,
                                            capi.REACTION_SQUARE, rows=rows)
    np.testing.assert_array_equal(h[rows], ho)
    assert hj_error(val[rows], hjo) <= TOL


def test_zero_coefficients_give_zero():
    mesh = dgfem.unit_square_mesh(8)
    ref = dgfem.ReferenceElement(3)
    h, _, _, val = device_nonlinear(mesh, ref, np.zeros(mesh.n_elements * ref.n_local),
                                    capi.REACTION_SQUARE)
    assert not h.any() and not val.any()


def test_jacobian_matches_finite_differences():
    """test_nonlinear.cpp:94-120 on the device: HJ against central differences of H."""
    mesh = dgfem.unit_square_mesh(4)
    ref = dgfem.ReferenceElement(1)
    nl = ref.n_local
    coef = 2.0 * problems.uniform01(2024, mesh.n_elements * nl) - 1.0
    _, _, _, val = device_nonlinear(mesh, ref, coef, capi.REACTION_SQUARE)
    delta = 1e-6
    for j in range(0, coef.size, 5):
        plus, minus = coef.copy(), coef.copy()
        plus[j] += delta
        minus[j] -= delta
        hp = device_nonlinear(mesh, ref, plus, capi.REACTION_SQUARE)[0].reshape(-1)
        hm = device_nonlinear(mesh, ref, minus, capi.REACTION_SQUARE)[0].reshape(-1)
        fd = (hp - hm) / (2 * delta)
        e = j // nl
        col = val[e][:, j % nl]
        rows = slice(e * nl, (e + 1) * nl)
        assert np.all(np.abs(col - fd[rows]) <= 1e-6 * np.maximum(1.0, np.abs(fd[rows])))
        others = np.delete(fd, np.arange(e * nl, (e + 1) * nl))
        assert np.abs(others).max() <= 1e-6


def test_bound_plan_reads_the_geometry_record():
    """P1 plan bound to the mesh (dgb_plan_bind_mesh builds the geometry record): the nonlinear
    kernel takes the vertices from the record instead of gathering nodes -- copies of the same
    coordinates, so H and HJ are bitwise what the unbound plan gives (ragged last chunk, jittered
    permuted mesh); a plan bound to a row shard keeps gathering."""
    import torch
    mesh = dgfem.unit_square_mesh(29, 0.2, 5, True, 6, 0)
    ref = dgfem.ReferenceElement(1)
    n = mesh.n_elements * ref.n_local
    coef = torch.from_numpy(2.0 * problems.uniform01(99, n) - 1.0).cuda()
    dm = dgfem.DeviceMesh(mesh)
    plan = dgfem.Plan(ref.view)
    h0, hj0 = plan.assemble_nonlinear(dm, coef, capi.REACTION_CUBIC)
    torch.cuda.synchronize()
    h0, v0 = h0.clone(), hj0.val.clone()
    for rows in ((0, mesh.n_elements), (0, mesh.n_elements // 2)):
        plan.bind_mesh(dm, *rows)
        h1, hj1 = plan.assemble_nonlinear(dm, coef, capi.REACTION_CUBIC)
        torch.cuda.synchronize()
        assert torch.equal(h0, h1) and torch.equal(v0, hj1.val)
