"""CPU: the product's host side (C++ behind the C-ABI) against the reference's own outputs:
mesh build (mesh.cpp:51-151), reference tables (reference.cpp:87-147), set_parameters
(assembly.cpp:483-506), error codes (errors.hpp:9-48); and the C-ABI surface itself."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1502_02941_b200 import capi, dgfem, problems

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def test_library_exports_every_header_symbol():
    """libdgfem_b200.so loads (no GPU needed) and exports every function include/*.h declares."""
    lib = C.CDLL(capi.LIB_PATH)
    declared = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            text = open(os.path.join(ROOT, "include", fn)).read()
            text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)  # drop comments
            declared |= set(re.findall(r"^[a-z][\w \*]*?\b(dgb_[a-z0-9_]+)\s*\(", text, re.M))
    assert len(declared) >= 20
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(capi.EXPORTED_SYMBOLS) <= declared
    assert capi.load().dgb_version().startswith(b"dgfem_b200")


def test_status_names_match_reference_error_codes():
    """1 + dgfem::ErrorCode, names as errors.cpp:5-27."""
    lib = capi.load()
    for status, name in enumerate(capi.STATUS_NAMES):
        assert lib.dgb_status_name(status).decode() == name
    assert lib.dgb_status_name(capi.STATUS_CUDA) == b"CudaError"


def test_set_parameters_per_method_defaults():
    """test_assembly.cpp:154-173."""
    p = dgfem.set_parameters(capi.SIPG, 1)
    assert (p.kappa, p.sigma_interior, p.sigma_boundary, p.degree) == (-1.0, 6.0, 12.0, 1)
    p = dgfem.set_parameters(capi.NIPG, 2)
    assert (p.kappa, p.sigma_interior, p.sigma_boundary) == (1.0, 1.0, 2.0)
    p = dgfem.set_parameters(capi.IIPG, 2)
    assert (p.kappa, p.sigma_interior, p.sigma_boundary) == (0.0, 18.0, 36.0)
    assert dgfem.set_parameters(capi.SIPG, 2).sigma_interior == 18.0
    with pytest.raises(dgfem.Error) as e:
        dgfem.set_parameters(capi.SIPG, 0)
    assert e.value.code == "InvalidArgument"


def test_config_parameters_override_sigma():
    """SURVEY.md finding 5: config 2 uses sigma = 18 for every method, boundary 2 sigma."""
    cfg = problems.CONFIGS[2]
    for m in cfg.methods:
        p = dgfem.config_parameters(cfg, m)
        assert (p.sigma_interior, p.sigma_boundary) == (18.0, 36.0)


def test_bsr_block_count_formula():
    for n in (1, 2, 7, 32):
        m = dgfem.unit_square_mesh(n)
        assert m.n_elements == 2 * n * n
        assert m.n_edges == 3 * n * n + 2 * n
        assert m.n_interior_edges == 3 * n * n - 2 * n
        assert capi.load().dgb_bsr_nnzb(m.n_elements, m.n_interior_edges) == 8 * n * n - 4 * n


# --------------------------------------------------------------------------- meshes
def _mesh_cases(z):
    return sorted({k.split("/")[0] for k in z.files if k.endswith("/out_edges")})


@pytest.mark.parametrize("name", _mesh_cases(np.load(os.path.join(GOLDEN, "meshes.npz"))))
def test_mesh_build_matches_reference(name):
    z = np.load(os.path.join(GOLDEN, "meshes.npz"))
    m = dgfem.build_mesh(z[f"{name}/in_nodes"], z[f"{name}/in_elements"],
                         z[f"{name}/in_dirichlet"], z[f"{name}/in_neumann"])
    for k, v in m.arrays().items():
        np.testing.assert_array_equal(v, z[f"{name}/out_{k}"].reshape(v.shape), err_msg=k)


def test_unit_square_generator_is_reproducible_and_matches_raw_rebuild():
    a = dgfem.unit_square_mesh(8, 0.2, 5, True, 6, 10)
    b = dgfem.build_mesh(**{k: v for k, v in zip(("nodes", "elements", "dirichlet", "neumann"),
                                                   (lambda r: (r["nodes"], r["elements"], r["dirichlet"], r["neumann"]))(a.raw()))})
    for k, v in a.arrays().items():
        np.testing.assert_array_equal(v, b.arrays()[k])
    c = dgfem.unit_square_mesh(8, 0.2, 5, True, 6, 10)
    np.testing.assert_array_equal(a.nodes, c.nodes)
    np.testing.assert_array_equal(a.elements, c.elements)
    # jitter is within +-0.2 h on interior nodes only; boundary nodes exact
    base = dgfem.unit_square_mesh(8)
    d = np.abs(a.nodes - base.nodes)
    assert d.max() <= 0.2 / 8 + 1e-15
    on_boundary = (base.nodes == 0.0) | (base.nodes == 1.0)
    assert np.all(d[on_boundary.any(axis=1)] == 0.0)


def test_config_mesh_sizes():
    """E, n_edges, I_int for every config (generator only, cheap)."""
    for idx in (1, 2, 5):
        cfg = problems.CONFIGS[idx]
        m = dgfem.config_mesh(cfg)
        n = cfg.n
        assert (m.n_elements, m.n_edges, m.n_interior_edges) == (2 * n * n, 3 * n * n + 2 * n,
                                                                 3 * n * n - 2 * n)


def _err_cases(z):
    return sorted({k.split("/")[0][4:] for k in z.files if k.startswith("err_") and k.endswith("/status")})


@pytest.mark.parametrize("name", _err_cases(np.load(os.path.join(GOLDEN, "meshes.npz"))))
def test_mesh_errors_match_reference(name):
    """Same ErrorCode and detail as dgfem::build_mesh for invalid input."""
    z = np.load(os.path.join(GOLDEN, "meshes.npz"))
    status, detail = int(z[f"err_{name}/status"]), int(z[f"err_{name}/detail"])
    assert status != 0
    with pytest.raises(dgfem.Error) as e:
        dgfem.build_mesh(z[f"err_{name}/nodes"], z[f"err_{name}/elements"],
                         z[f"err_{name}/dirichlet"], z[f"err_{name}/neumann"])
    assert e.value.status == status, (e.value.code, capi.STATUS_NAMES[status])
    assert e.value.detail == detail


# --------------------------------------------------------------------------- tables
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_reference_tables_match_reference_bitwise(k):
    z = np.load(os.path.join(GOLDEN, "tables.npz"))
    for qo in (0, 2 * k + 1):
        t = dgfem.ReferenceElement(k, qo).tables()
        for name, v in t.items():
            np.testing.assert_array_equal(np.asarray(v), z[f"k{k}_q{qo}_{name}"], err_msg=f"{qo} {name}")


def test_reference_config_quadrature_sizes():
    """SURVEY.md finding 2: quad_order = 2k+1 gives k+1 edge points, 6/7/16/19 volume points."""
    for k, nq in zip((1, 2, 3, 4), (6, 7, 16, 19)):
        r = dgfem.ReferenceElement(k, 2 * k + 1)
        assert (r.nq_vol, r.nq_edge, r.n_local) == (nq, k + 1, (k + 1) * (k + 2) // 2)


def test_unsupported_degree():
    with pytest.raises(dgfem.Error) as e:
        dgfem.ReferenceElement(5)
    assert e.value.code == "UnsupportedDegree" and e.value.detail == 5


def test_orthonormal_basis_mass_is_identity():
    """reference.hpp:18-21: the reference mass matrix is the identity."""
    for k in (1, 2, 3, 4):
        t = dgfem.ReferenceElement(k).tables()
        nl = t["n_local"]
        phi = t["phi"].reshape(-1, nl)
        M = (phi * t["vol_w"][:, None]).T @ phi
        assert np.abs(M - np.eye(nl)).max() < 1e-13


def test_assemble_terms_rejects_bad_mask_before_any_device_work():
    """dgb_assemble_terms validates its term mask on the host (no GPU needed)."""
    from paper_1502_02941_b200 import problems
    lib = capi.load()
    spec = problems.registry_get("smooth-sine")
    params = capi.Params()
    st = lib.dgb_assemble_terms(None, None, C.byref(spec.c), C.byref(params), 9, None, None, None)
    assert capi.STATUS_NAMES[st] == "InvalidArgument"
    assert b"term mask" in lib.dgb_last_error_message()
