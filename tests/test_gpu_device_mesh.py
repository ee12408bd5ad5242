"""GPU: build_mesh and uniform_refine on the device (mesh.cpp:51-187)
against the reference's own outputs (tests/golden/meshes.npz, refine.npz): every array
bit-identical, every error with the reference's code and detail."""
import os

import numpy as np
import pytest

from paper_1502_02941_b200 import capi, dgfem, problems

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
KEYS = ("nodes", "elements", "edges", "edge_kind", "edge_elements", "element_edges")


def mesh_names(z):
    return sorted({k.split("/")[0] for k in z.files if k.endswith("/out_nodes")})


@pytest.mark.parametrize("name", mesh_names(np.load(os.path.join(GOLDEN, "meshes.npz"))))
def test_device_build_matches_reference(name):
    z = np.load(os.path.join(GOLDEN, "meshes.npz"))
    m = dgfem.device_build_mesh(z[f"{name}/in_nodes"], z[f"{name}/in_elements"],
                                z[f"{name}/in_dirichlet"], z[f"{name}/in_neumann"])
    a = m.arrays()
    for k in KEYS:
        np.testing.assert_array_equal(a[k].reshape(-1), z[f"{name}/out_{k}"].reshape(-1), err_msg=k)
    assert m.n_interior_edges == int((z[f"{name}/out_edge_elements"].reshape(-1, 2)[:, 1] >= 0).sum())


def error_names(z):
    return sorted({k.split("/")[0][4:] for k in z.files if k.startswith("err_")})


@pytest.mark.parametrize("name", error_names(np.load(os.path.join(GOLDEN, "meshes.npz"))))
def test_device_build_errors_match_reference(name):
    z = np.load(os.path.join(GOLDEN, "meshes.npz"))
    p = f"err_{name}"
    status, detail = int(z[f"{p}/status"]), int(z[f"{p}/detail"])
    args = [z[f"{p}/nodes"], z[f"{p}/elements"], z[f"{p}/dirichlet"], z[f"{p}/neumann"]]
    if status == 0:
        dgfem.device_build_mesh(*args)
        return
    with pytest.raises(dgfem.Error) as e:
        dgfem.device_build_mesh(*args)
    assert e.value.status == status and e.value.detail == detail, (e.value.code, e.value.detail)


@pytest.mark.parametrize("sides", [0, 2 | 8])
def test_device_refine_matches_reference(sides):
    z = np.load(os.path.join(GOLDEN, "refine.npz"))
    b = f"s{sides}_l0"
    edges, kind = z[f"{b}/edges"].reshape(-1, 2), z[f"{b}/edge_kind"]
    m = dgfem.device_build_mesh(z[f"{b}/nodes"], z[f"{b}/elements"], edges[kind == 1], edges[kind == 2])
    for _ in range(4):
        m = m.refine()
    a = m.arrays()
    for k in KEYS:
        np.testing.assert_array_equal(a[k].reshape(-1), z[f"s{sides}_l4/{k}"].reshape(-1), err_msg=k)


def test_device_build_config4_size_equals_host_build():
    """Config 4's mesh (2048^2 x 2 triangles, permuted numbering): the device build of the raw
    input equals the host builder's (itself pinned to the reference) array for array."""
    cfg = problems.CONFIGS[4]
    host = dgfem.config_mesh(cfg)
    raw = host.raw()
    dev = dgfem.device_build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
    a, h = dev.arrays(), host.arrays()
    for k in KEYS:
        assert np.array_equal(a[k].reshape(-1), np.asarray(h[k]).reshape(-1)), k


def test_assembly_on_device_built_mesh_is_identical():
    cfg = problems.CONFIGS[2]
    host = dgfem.unit_square_mesh(32, 0.2, 5, True, 6)
    raw = host.raw()
    dev = dgfem.device_build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(2)
    p = dgfem.config_parameters(cfg, capi.SIPG)
    plan = dgfem.Plan(ref.view)
    dm, dp = dgfem.DeviceMesh(host), dgfem.DeviceProblem(spec)
    a = plan.assemble(dm, dp, p, plan.allocate(dm))
    b = plan.assemble(dev, dp, p, plan.allocate(dm))
    for x, y in ((a.row_ptr, b.row_ptr), (a.col, b.col), (a.val, b.val), (a.rhs, b.rhs)):
        assert bool((x == y).all())
