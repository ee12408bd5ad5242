"""ctypes mirror of include/dgfem_b200.h (the C-ABI drop-in boundary).

Only type definitions and the loader live here; the user-facing Python API that mirrors the
reference's `dgfem::assemble_all` interface is in `dgfem.py`.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdgfem_b200.so")

# --- enums (dgfem_b200.h) ---------------------------------------------------------------
EDGE_INTERIOR, EDGE_DIRICHLET, EDGE_NEUMANN = 0, 1, 2
FIELD_CONSTANT, FIELD_PER_ELEMENT, FIELD_FUNCTION = 0, 1, 2
FN_SIN_SIN, FN_TANH_LAYER, FN_GAUSSIAN, FN_AFFINE, FN_STEP_Y = 1, 2, 3, 4, 5
MODE_VALUE, MODE_SOURCE, MODE_FLUX_X, MODE_SOURCE_SQUARE = 0, 1, 2, 3
VEC_CONSTANT, VEC_AFFINE, VEC_TRIG = 0, 1, 2
SIPG, NIPG, IIPG = 0, 1, 2
INFLOW_ERROR, INFLOW_DROP = 0, 1

# 1 + dgfem::ErrorCode (errors.hpp:9-27)
STATUS_NAMES = [
    "Ok", "InvalidTopology", "InvalidBoundarySpec", "NonManifold", "DegenerateElement",
    "UnsupportedDegree", "InvalidIndex", "DimensionMismatch", "SingularMatrix",
    "SolveAccuracy", "InflowOnNeumann", "NonPositiveDiffusion", "InvalidReaction",
    "NoExactSolution", "UnknownProblem", "UnknownMethod", "IoFailure", "InvalidArgument",
]
STATUS_CUDA = 100


class MeshArrays(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int32), ("n_elements", C.c_int32), ("n_edges", C.c_int32),
        ("n_interior_edges", C.c_int32),
        ("nodes", C.c_void_p), ("elements", C.c_void_p), ("edges", C.c_void_p),
        ("edge_kind", C.c_void_p), ("edge_elements", C.c_void_p),
        ("element_edges", C.c_void_p),
    ]


class ReferenceTables(C.Structure):
    _fields_ = [
        ("degree", C.c_int32), ("n_local", C.c_int32), ("nq_vol", C.c_int32),
        ("nq_edge", C.c_int32),
        ("vol_x", C.c_void_p), ("vol_y", C.c_void_p), ("vol_w", C.c_void_p),
        ("edge_t", C.c_void_p), ("edge_w", C.c_void_p),
        ("phi", C.c_void_p), ("dphi", C.c_void_p),
        ("edge_phi", C.c_void_p), ("edge_dphi", C.c_void_p),
    ]


class ScalarField(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("fn", C.c_int32), ("mode", C.c_int32), ("pad_", C.c_int32),
        ("value", C.c_double), ("p", C.c_double * 4), ("q", C.c_double * 4),
        ("per_element", C.c_void_p),
    ]


class VectorField(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("p", C.c_double * 6)]


class Problem(C.Structure):
    _fields_ = [
        ("diffusion", ScalarField), ("advection", VectorField),
        ("linear_reaction", ScalarField), ("source", ScalarField),
        ("dirichlet", ScalarField), ("neumann", ScalarField),
    ]


class Params(C.Structure):
    _fields_ = [
        ("method", C.c_int32), ("degree", C.c_int32), ("kappa", C.c_double),
        ("sigma_interior", C.c_double), ("sigma_boundary", C.c_double),
        ("neumann_inflow", C.c_int32), ("pad_", C.c_int32),
    ]


class Bsr(C.Structure):
    _fields_ = [
        ("n_block_rows", C.c_int32), ("block_dim", C.c_int32), ("nnzb", C.c_int64),
        ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p),
    ]


class Reaction(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32)]


REACTION_ZERO, REACTION_LINEAR, REACTION_SQUARE, REACTION_CUBIC = 0, 1, 2, 3
TERM_DIFFUSION, TERM_CONVECTION, TERM_REACTION, TERM_ALL = 1, 2, 4, 7
PRECOND_BLOCK_JACOBI, PRECOND_BLOCK_SGS = 0, 1


class SolveOptions(C.Structure):
    _fields_ = [("tolerance_scale", C.c_double), ("max_iterations", C.c_int32),
                ("restart", C.c_int32), ("preconditioner", C.c_int32), ("pad_", C.c_int32)]


class SolveInfo(C.Structure):
    _fields_ = [("defect_norm2", C.c_double), ("defect_norm_inf", C.c_double),
                ("bound", C.c_double), ("iterations", C.c_int32), ("restarts", C.c_int32)]


class NewtonConfig(C.Structure):
    _fields_ = [("max_iterations", C.c_int32), ("use_legacy_check", C.c_int32),
                ("residual_tolerance", C.c_double), ("step_tolerance", C.c_double),
                ("legacy_check", C.c_double)]


class NewtonReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32),
                ("final_residual", C.c_double), ("residual_history", C.c_void_p),
                ("linear_iterations", C.c_int32), ("pad_", C.c_int32)]


def _declare(lib: C.CDLL) -> C.CDLL:
    P = C.POINTER
    vp = C.c_void_p
    sigs = {
        "dgb_status_name": (C.c_char_p, [C.c_int]),
        "dgb_last_error_message": (C.c_char_p, []),
        "dgb_last_error_detail": (C.c_longlong, []),
        "dgb_version": (C.c_char_p, []),
        "dgb_mesh_build": (C.c_int, [vp, C.c_int32, vp, C.c_int32, vp, C.c_int32, vp,
                                     C.c_int32, P(vp)]),
        "dgb_mesh_unit_square": (C.c_int, [C.c_int32, C.c_double, C.c_uint64, C.c_int32,
                                           C.c_uint64, C.c_int32, P(vp)]),
        "dgb_mesh_rectangle": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                         C.c_uint64, C.c_int32, C.c_uint64, C.c_int32, P(vp)]),
        "dgb_mesh_view": (C.c_int, [vp, P(MeshArrays)]),
        "dgb_mesh_raw": (C.c_int, [vp, P(vp), P(C.c_int32), P(vp), P(C.c_int32), P(vp),
                                   P(C.c_int32), P(vp), P(C.c_int32)]),
        "dgb_mesh_free": (None, [vp]),
        "dgb_reference_create": (C.c_int, [C.c_int32, C.c_int32, P(vp)]),
        "dgb_reference_view": (C.c_int, [vp, P(ReferenceTables)]),
        "dgb_reference_free": (None, [vp]),
        "dgb_set_parameters": (C.c_int, [C.c_int32, C.c_int32, P(Params)]),
        "dgb_bsr_nnzb": (C.c_int64, [C.c_int32, C.c_int32]),
        "dgb_plan_create": (C.c_int, [P(ReferenceTables), C.c_int32, P(vp)]),
        "dgb_plan_destroy": (None, [vp]),
        "dgb_assemble": (C.c_int, [vp, P(MeshArrays), P(Problem), P(Params), P(Bsr), vp, vp]),
        "dgb_assemble_terms": (C.c_int, [vp, P(MeshArrays), P(Problem), P(Params), C.c_int32, P(Bsr),
                                         vp, vp]),
        "dgb_plan_status": (C.c_int, [vp, vp]),
        "dgb_plan_set_kernel_events": (C.c_int, [vp, vp, vp]),
        "dgb_plan_bind_mesh": (C.c_int, [vp, P(MeshArrays), C.c_int32, C.c_int32, vp]),
        "dgb_plan_unbind_mesh": (C.c_int, [vp]),
        "dgb_plan_launch_count": (C.c_int32, [vp]),
        "dgb_plan_set_option": (C.c_int, [vp, C.c_int32, C.c_int32]),
        "dgb_spmv": (C.c_int, [P(Bsr), vp, vp, vp]),
        "dgb_assemble_rows": (C.c_int, [vp, P(MeshArrays), P(Problem), P(Params), C.c_int32,
                                        C.c_int32, P(Bsr), vp, vp]),
        "dgb_count_blocks_host": (C.c_int64, [P(MeshArrays), C.c_int32, C.c_int32]),
        "dgb_assemble_all_host": (C.c_int, [P(MeshArrays), P(ReferenceTables), P(Problem),
                                            P(Params), C.c_int32, P(Bsr), vp]),
        "dgb_assemble_nonlinear": (C.c_int, [vp, P(MeshArrays), vp, C.c_int64, P(Reaction), vp,
                                             P(Bsr), vp]),
        "dgb_assemble_nonlinear_host": (C.c_int, [P(MeshArrays), P(ReferenceTables), vp,
                                                  C.c_int64, P(Reaction), C.c_int32, vp, P(Bsr)]),
        "dgb_device_mesh_build": (C.c_int, [vp, C.c_int32, vp, C.c_int32, vp, C.c_int32, vp,
                                            C.c_int32, C.c_int32, P(vp), vp]),
        "dgb_device_mesh_refine": (C.c_int, [vp, P(vp), vp]),
        "dgb_device_mesh_view": (C.c_int, [vp, P(MeshArrays)]),
        "dgb_device_mesh_free": (None, [vp]),
        "dgb_device_mesh_copy_to_host": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
        "dgb_assemble_batch": (C.c_int, [vp, P(MeshArrays), P(Problem), P(Params), C.c_int32,
                                         C.c_int32, C.c_int32, P(Bsr), P(vp), vp]),
        "dgb_l2_quad_order": (C.c_int32, [C.c_int32, C.c_int32]),
        "dgb_l2_error": (C.c_int, [vp, P(MeshArrays), vp, C.c_int64, P(ScalarField), vp, vp]),
        "dgb_project": (C.c_int, [vp, P(MeshArrays), P(ScalarField), vp, vp]),
        "dgb_eval_solution": (C.c_int, [vp, C.c_int32, C.c_int32, C.c_int64, vp, vp, vp, vp, vp]),
        "dgb_solve_options_default": (None, [P(SolveOptions)]),
        "dgb_newton_config_default": (None, [P(NewtonConfig)]),
        "dgb_solve": (C.c_int, [P(Bsr), vp, vp, P(SolveOptions), P(SolveInfo), vp]),
        "dgb_newton_solve": (C.c_int, [vp, P(MeshArrays), P(Bsr), vp, P(Reaction), P(NewtonConfig),
                                       P(SolveOptions), vp, P(NewtonReport), vp]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


EXPORTED_SYMBOLS = [
    "dgb_status_name", "dgb_last_error_message", "dgb_last_error_detail", "dgb_version",
    "dgb_mesh_build", "dgb_mesh_unit_square", "dgb_mesh_view", "dgb_mesh_raw",
    "dgb_mesh_free", "dgb_reference_create", "dgb_reference_view", "dgb_reference_free",
    "dgb_set_parameters", "dgb_bsr_nnzb", "dgb_plan_create", "dgb_plan_destroy",
    "dgb_assemble", "dgb_assemble_terms", "dgb_plan_status", "dgb_plan_set_kernel_events",
    "dgb_plan_bind_mesh", "dgb_plan_unbind_mesh", "dgb_plan_launch_count", "dgb_plan_set_option", "dgb_spmv", "dgb_assemble_all_host",
    "dgb_mesh_rectangle", "dgb_assemble_rows", "dgb_count_blocks_host",
    "dgb_assemble_nonlinear", "dgb_assemble_nonlinear_host",
    "dgb_solve_options_default", "dgb_newton_config_default", "dgb_solve", "dgb_newton_solve",
    "dgb_l2_quad_order", "dgb_l2_error", "dgb_project", "dgb_eval_solution",
    "dgb_device_mesh_build", "dgb_device_mesh_refine", "dgb_device_mesh_view",
    "dgb_device_mesh_free", "dgb_device_mesh_copy_to_host", "dgb_assemble_batch",
]
OPTION_FORCE_GENERIC_KERNEL = 1
OPTION_MIN_BLOCKS = 2
OPTION_L2_POLICY = 3
OPTION_BATCH_FUSE = 4
OPTION_WARP_SPECIALIZED = 5
OPTION_P1_PIPELINE = 6
OPTION_L2_CARVEOUT_MB = 7
OPTION_GEOMETRY_CACHE = 8
OPTION_PROFILE_ABLATE = 1000  # diagnostics only: results are wrong while set

_lib = None


def load() -> C.CDLL:
    """Loads the in-tree libdgfem_b200.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the CUDA extension is required; there is no CPU fallback)")
        _lib = _declare(C.CDLL(LIB_PATH))
    return _lib
