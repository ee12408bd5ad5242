"""Python mirror of the reference's assembly interface, over the C-ABI (include/dgfem_b200.h).

Names and argument meaning follow /root/reference/proj/include/dgfem/assembly.hpp:
`set_parameters(method, degree)`, `assemble_all(mesh, ref, problem, params)`; errors raise
`Error` with the reference's `ErrorCode` name and `detail` (errors.hpp:35-48).  The device
arrays are torch CUDA tensors (torch is plumbing: memory, streams, events); the work is done
by the sm_100a kernels in libdgfem_b200.so.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import capi
from .capi import Bsr, MeshArrays, Params, ReferenceTables
from .problems import ProblemSpec


class Error(RuntimeError):
    """dgfem::Error: `code` is the ErrorCode name, `detail` the offending index or -1."""

    def __init__(self, status: int, message: str, detail: int):
        super().__init__(message)
        self.status = status
        self.code = capi.STATUS_NAMES[status] if 0 <= status < len(capi.STATUS_NAMES) else (
            "CudaError" if status == capi.STATUS_CUDA else str(status))
        self.detail = detail


def _check(status: int) -> None:
    if status != 0:
        lib = capi.load()
        raise Error(status, lib.dgb_last_error_message().decode(), int(lib.dgb_last_error_detail()))


_DT = {C.c_double: np.float64, C.c_int32: np.int32, C.c_uint8: np.uint8}


def _np(ptr, n, ctype, shape):
    if n == 0 or not ptr:
        return np.zeros(shape, dtype=_DT[ctype])
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(n,)).reshape(shape)


# ------------------------------------------------------------------------------ mesh
class Mesh:
    """Host mesh (dgfem::Mesh, mesh.hpp:37-49) built by the C++ host library."""

    def __init__(self, handle: C.c_void_p):
        self._lib = capi.load()
        self._h = handle
        v = MeshArrays()
        _check(self._lib.dgb_mesh_view(handle, C.byref(v)))
        self.view = v
        self.n_nodes, self.n_elements, self.n_edges = v.n_nodes, v.n_elements, v.n_edges
        self.n_interior_edges = v.n_interior_edges
        self.nodes = _np(v.nodes, 2 * v.n_nodes, C.c_double, (v.n_nodes, 2))
        self.elements = _np(v.elements, 3 * v.n_elements, C.c_int32, (v.n_elements, 3))
        self.edges = _np(v.edges, 2 * v.n_edges, C.c_int32, (v.n_edges, 2))
        self.edge_kind = _np(v.edge_kind, v.n_edges, C.c_uint8, (v.n_edges,))
        self.edge_elements = _np(v.edge_elements, 2 * v.n_edges, C.c_int32, (v.n_edges, 2))
        self.element_edges = _np(v.element_edges, 3 * v.n_elements, C.c_int32, (v.n_elements, 3))

    def arrays(self) -> dict:
        """The six mesh arrays as numpy (views into the C++ storage)."""
        return {k: getattr(self, k) for k in ("nodes", "elements", "edges", "edge_kind",
                                              "edge_elements", "element_edges")}

    def raw(self) -> dict:
        """Input that produced the mesh (for feeding the reference's build_mesh)."""
        nodes, elements, dirichlet, neumann = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        nn, ne, nd, nm = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(self._lib.dgb_mesh_raw(self._h, C.byref(nodes), C.byref(nn), C.byref(elements),
                                      C.byref(ne), C.byref(dirichlet), C.byref(nd),
                                      C.byref(neumann), C.byref(nm)))
        return {
            "nodes": _np(nodes.value, 2 * nn.value, C.c_double, (nn.value, 2)).copy(),
            "elements": _np(elements.value, 3 * ne.value, C.c_int32, (ne.value, 3)).copy(),
            "dirichlet": (_np(dirichlet.value, 2 * nd.value, C.c_int32, (nd.value, 2)).copy()
                          if nd.value else np.zeros((0, 2), np.int32)),
            "neumann": (_np(neumann.value, 2 * nm.value, C.c_int32, (nm.value, 2)).copy()
                        if nm.value else np.zeros((0, 2), np.int32)),
        }

    def __del__(self):
        try:
            self._lib.dgb_mesh_free(self._h)
        except Exception:
            pass


def build_mesh(nodes, elements, dirichlet, neumann) -> Mesh:
    """dgfem::build_mesh (mesh.hpp:62-65)."""
    lib = capi.load()
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    elements = np.ascontiguousarray(elements, dtype=np.int32)
    dirichlet = np.ascontiguousarray(dirichlet, dtype=np.int32).reshape(-1, 2)
    neumann = np.ascontiguousarray(neumann, dtype=np.int32).reshape(-1, 2)
    h = C.c_void_p()
    _check(lib.dgb_mesh_build(nodes.ctypes.data, nodes.shape[0], elements.ctypes.data,
                              elements.shape[0], dirichlet.ctypes.data, dirichlet.shape[0],
                              neumann.ctypes.data, neumann.shape[0], C.byref(h)))
    return Mesh(h)


def unit_square_mesh(n: int, jitter: float = 0.0, jitter_seed: int = 0, permute: bool = False,
                     permute_seed: int = 0, neumann_sides: int = 0) -> Mesh:
    """The BASELINE.json structured meshes (see dgb_mesh_unit_square)."""
    lib = capi.load()
    h = C.c_void_p()
    _check(lib.dgb_mesh_unit_square(n, jitter, jitter_seed, int(permute), permute_seed,
                                    neumann_sides, C.byref(h)))
    return Mesh(h)


def rectangle_mesh(nx: int, ny: int, lx: float, ly: float, jitter: float = 0.0,
                   jitter_seed: int = 0, permute: bool = False, permute_seed: int = 0,
                   neumann_sides: int = 0) -> Mesh:
    """dgb_mesh_rectangle: the same construction on [0, lx] x [0, ly]."""
    lib = capi.load()
    h = C.c_void_p()
    _check(lib.dgb_mesh_rectangle(nx, ny, lx, ly, jitter, jitter_seed, int(permute),
                                  permute_seed, neumann_sides, C.byref(h)))
    return Mesh(h)


def config_mesh(cfg, strips: int = 1) -> Mesh:
    """Config mesh; strips > 1 gives the weak-scaling global mesh ([0, strips] x [0, 1], i.e.
    `strips` config-sized squares side by side).  strips = 1 is the config's unit square."""
    from .problems import SEED_JITTER, SEED_PERMUTE
    if strips == 1:
        return unit_square_mesh(cfg.n, cfg.jitter, SEED_JITTER, cfg.permute, SEED_PERMUTE,
                                cfg.neumann_sides)
    return rectangle_mesh(strips * cfg.n, cfg.n, float(strips), 1.0, cfg.jitter, SEED_JITTER,
                          cfg.permute, SEED_PERMUTE, cfg.neumann_sides)


# ------------------------------------------------------------------------------ reference
class ReferenceElement:
    """dgfem::ReferenceElement(degree, quad_order) (reference.hpp:22-77)."""

    def __init__(self, degree: int, quad_order: int = 0):
        self._lib = capi.load()
        h = C.c_void_p()
        _check(self._lib.dgb_reference_create(degree, quad_order, C.byref(h)))
        self._h = h
        self.quad_order = quad_order
        v = ReferenceTables()
        _check(self._lib.dgb_reference_view(h, C.byref(v)))
        self.view = v
        self.degree, self.n_local = v.degree, v.n_local
        self.nq_vol, self.nq_edge = v.nq_vol, v.nq_edge

    def tables(self) -> dict:
        v, nl, nq, ne = self.view, self.n_local, self.nq_vol, self.nq_edge

        def arr(ptr, n):
            return _np(ptr, n, C.c_double, (n,)).copy()
        return {
            "degree": self.degree, "n_local": nl, "nq_vol": nq, "nq_edge": ne,
            "vol_x": arr(v.vol_x, nq), "vol_y": arr(v.vol_y, nq), "vol_w": arr(v.vol_w, nq),
            "edge_t": arr(v.edge_t, ne), "edge_w": arr(v.edge_w, ne),
            "phi": arr(v.phi, nq * nl), "dphi": arr(v.dphi, nq * nl * 2),
            "edge_phi": arr(v.edge_phi, 6 * ne * nl),
            "edge_dphi": arr(v.edge_dphi, 6 * ne * nl * 2),
        }

    def __del__(self):
        try:
            self._lib.dgb_reference_free(self._h)
        except Exception:
            pass


def tables_struct(t: dict) -> ReferenceTables:
    """A ReferenceTables view over a dict of numpy tables (e.g. the reference's own)."""
    v = ReferenceTables()
    v.degree, v.n_local, v.nq_vol, v.nq_edge = t["degree"], t["n_local"], t["nq_vol"], t["nq_edge"]
    for k in ("vol_x", "vol_y", "vol_w", "edge_t", "edge_w", "phi", "dphi", "edge_phi",
              "edge_dphi"):
        setattr(v, k, np.ascontiguousarray(t[k], dtype=np.float64).ctypes.data)
    return v


# ------------------------------------------------------------------------------ params
def set_parameters(method: int, degree: int, neumann_inflow: int = capi.INFLOW_ERROR) -> Params:
    """dgfem::set_parameters (assembly.cpp:483-506)."""
    p = Params()
    _check(capi.load().dgb_set_parameters(method, degree, C.byref(p)))
    p.neumann_inflow = neumann_inflow
    return p


def config_parameters(cfg, method: int) -> Params:
    """Config parameters: sigma override for every method, boundary = 2 sigma
    (SURVEY.md finding 5; the reference's --penalty, cli.cpp:130-136)."""
    p = set_parameters(method, cfg.degree, cfg.neumann_inflow)
    p.sigma_interior = cfg.sigma
    p.sigma_boundary = 2.0 * cfg.sigma
    return p


# ------------------------------------------------------------------------------ device
class DeviceMesh:
    """Mesh arrays resident in HBM (torch CUDA tensors) + the C view over them."""

    def __init__(self, mesh: Mesh, device: int = 0):
        import torch
        dev = torch.device("cuda", device)
        self.n_elements, self.n_interior_edges = mesh.n_elements, mesh.n_interior_edges
        self.t = {k: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                  for k, a in mesh.arrays().items()}
        v = MeshArrays()
        v.n_nodes, v.n_elements, v.n_edges = mesh.n_nodes, mesh.n_elements, mesh.n_edges
        v.n_interior_edges = mesh.n_interior_edges
        for k, a in self.t.items():
            setattr(v, k, a.data_ptr())
        self.view = v


class DeviceProblem:
    """A problem descriptor whose per-element fields point at device copies."""

    def __init__(self, spec: ProblemSpec, device: int = 0):
        import torch
        self.spec = spec
        self.c = type(spec.c).from_buffer_copy(spec.c)
        self.t = {}
        for name, arr in spec.per_element.items():
            t = torch.from_numpy(arr).to(torch.device("cuda", device))
            self.t[name] = t
            getattr(self.c, name).per_element = t.data_ptr()


@dataclass
class BsrSystem:
    """Assembled K (BSR, sorted block columns, nl x nl row-major blocks) and F, on device."""
    row_ptr: "object"
    col: "object"
    val: "object"
    rhs: "object"
    block_dim: int

    def struct(self) -> Bsr:
        b = Bsr()
        b.n_block_rows = self.row_ptr.shape[0] - 1
        b.block_dim = self.block_dim
        b.nnzb = self.col.shape[0]
        b.row_ptr, b.col, b.val = self.row_ptr.data_ptr(), self.col.data_ptr(), self.val.data_ptr()
        return b


class Plan:
    """dgb_plan: device-resident contraction tensors for one ReferenceElement."""

    def __init__(self, tables: ReferenceTables, device: int = 0):
        self._lib = capi.load()
        h = C.c_void_p()
        _check(self._lib.dgb_plan_create(C.byref(tables), device, C.byref(h)))
        self._h = h
        self.device = device
        self.n_local = tables.n_local

    def set_option(self, option: int, value: int) -> None:
        _check(self._lib.dgb_plan_set_option(self._h, option, value))

    def bind_mesh(self, dmesh: "DeviceMesh", row_begin: int = 0, row_end: int | None = None,
                  stream=None) -> None:
        """dgb_plan_bind_mesh: compute the BSR pattern once for this mesh / row range."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        h = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        end = dmesh.n_elements if row_end is None else row_end
        _check(self._lib.dgb_plan_bind_mesh(self._h, C.byref(dmesh.view), row_begin, end,
                                            C.c_void_p(h)))

    def set_generic(self, on: bool = True) -> None:
        """Force the generic block-row kernel (testing)."""
        _check(self._lib.dgb_plan_set_option(self._h, capi.OPTION_FORCE_GENERIC_KERNEL, int(on)))

    def allocate(self, dmesh: DeviceMesh) -> BsrSystem:
        import torch
        dev = torch.device("cuda", self.device)
        nl, E = self.n_local, dmesh.n_elements
        nnzb = self._lib.dgb_bsr_nnzb(E, dmesh.n_interior_edges)
        return BsrSystem(torch.empty(E + 1, dtype=torch.int32, device=dev),
                         torch.empty(nnzb, dtype=torch.int32, device=dev),
                         torch.empty((nnzb, nl, nl), dtype=torch.float64, device=dev),
                         torch.empty((E, nl), dtype=torch.float64, device=dev), nl)

    def assemble(self, dmesh: DeviceMesh, dproblem: DeviceProblem, params: Params,
                 out: BsrSystem, stream=None, check: bool = True) -> BsrSystem:
        """Enqueues the assembly on `stream` (torch stream or raw handle; default: torch's
        current stream).  check=True waits and raises the reference's error, if any."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        b = out.struct()
        _check(self._lib.dgb_assemble(self._h, C.byref(dmesh.view), C.byref(dproblem.c),
                                      C.byref(params), C.byref(b), out.rhs.data_ptr(),
                                      C.c_void_p(handle)))
        if check:
            _check(self._lib.dgb_plan_status(self._h, C.c_void_p(handle)))
        return out

    def assemble_terms(self, dmesh: DeviceMesh, dproblem: DeviceProblem, params: Params,
                       terms: int, out: BsrSystem, stream=None, check: bool = True) -> BsrSystem:
        """dgb_assemble_terms: K of the selected terms only (capi.TERM_* mask), e.g. the
        reference's `assemble_diffusion(...).D` for capi.TERM_DIFFUSION."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        b = out.struct()
        _check(self._lib.dgb_assemble_terms(self._h, C.byref(dmesh.view), C.byref(dproblem.c),
                                            C.byref(params), terms, C.byref(b),
                                            out.rhs.data_ptr(), C.c_void_p(handle)))
        if check:
            _check(self._lib.dgb_plan_status(self._h, C.c_void_p(handle)))
        return out

    def assemble_nonlinear(self, dmesh: DeviceMesh, coef, reaction: int, h=None, hj=None,
                           stream=None):
        """dgb_assemble_nonlinear on device tensors: H [E, nl] and the block-diagonal HJ
        (BsrSystem with rhs=None) for `coef` [E * nl] and the reaction kind (capi.REACTION_*)."""
        import torch
        dev = torch.device("cuda", self.device)
        nl, E = self.n_local, dmesh.n_elements
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        if h is None:
            h = torch.empty((E, nl), dtype=torch.float64, device=dev)
        if hj is None:
            hj = BsrSystem(torch.empty(E + 1, dtype=torch.int32, device=dev),
                           torch.empty(E, dtype=torch.int32, device=dev),
                           torch.empty((E, nl, nl), dtype=torch.float64, device=dev), None, nl)
        r = capi.Reaction()
        r.kind = reaction
        b = hj.struct()
        _check(self._lib.dgb_assemble_nonlinear(self._h, C.byref(dmesh.view), coef.data_ptr(),
                                                coef.numel(), C.byref(r), h.data_ptr(),
                                                C.byref(b), C.c_void_p(handle)))
        return h, hj

    def spmv(self, system: BsrSystem, x, y, stream=None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        b = system.struct()
        _check(self._lib.dgb_spmv(C.byref(b), x.data_ptr(), y.data_ptr(), C.c_void_p(handle)))
        return y

    def __del__(self):
        try:
            self._lib.dgb_plan_destroy(self._h)
        except Exception:
            pass


def assemble_all(mesh: Mesh, ref: ReferenceElement, problem: ProblemSpec, params: Params,
                 device: int = 0, generic: bool = False) -> BsrSystem:
    """`dgfem::assemble_all(mesh, ref, problem, params)` + `stiffness()` on the GPU: returns
    K (BSR) and F as device tensors.  Raises Error like the reference."""
    plan = Plan(ref.view, device)
    if generic:
        plan.set_generic(True)
    dmesh = DeviceMesh(mesh, device)
    dprob = DeviceProblem(problem, device)
    out = plan.allocate(dmesh)
    return plan.assemble(dmesh, dprob, params, out)


def assemble_all_host(mesh: Mesh, tables: ReferenceTables, problem: ProblemSpec,
                      params: Params, device: int = 0):
    """The host-buffer one-shot C entry point (dgb_assemble_all_host): numpy in, numpy out."""
    lib = capi.load()
    nl = tables.n_local
    E = mesh.n_elements
    nnzb = lib.dgb_bsr_nnzb(E, mesh.n_interior_edges)
    row_ptr = np.zeros(E + 1, np.int32)
    col = np.zeros(nnzb, np.int32)
    val = np.zeros((nnzb, nl, nl))
    rhs = np.zeros((E, nl))
    b = Bsr()
    b.n_block_rows, b.block_dim, b.nnzb = E, nl, nnzb
    b.row_ptr, b.col, b.val = row_ptr.ctypes.data, col.ctypes.data, val.ctypes.data
    _check(lib.dgb_assemble_all_host(C.byref(mesh.view), C.byref(tables), C.byref(problem.c),
                                     C.byref(params), device, C.byref(b), rhs.ctypes.data))
    return row_ptr, col, val, rhs


def assemble_nonlinear(coef, mesh: Mesh, ref: ReferenceElement, reaction: int, device: int = 0):
    """`dgfem::assemble_nonlinear(coef, mesh, ref, reaction)` (nonlinear.cpp:11-107) through
    the host-buffer entry point: numpy in, (h [E*nl], (row_ptr, col, val [E, nl, nl])) out --
    HJ as its block diagonal (BSR, one block per element)."""
    lib = capi.load()
    coef = np.ascontiguousarray(coef, dtype=np.float64)
    nl, E = ref.n_local, mesh.n_elements
    h = np.zeros(E * nl)
    row_ptr = np.zeros(E + 1, np.int32)
    col = np.zeros(E, np.int32)
    val = np.zeros((E, nl, nl))
    b = Bsr()
    b.n_block_rows, b.block_dim, b.nnzb = E, nl, E
    b.row_ptr, b.col, b.val = row_ptr.ctypes.data, col.ctypes.data, val.ctypes.data
    r = capi.Reaction()
    r.kind = reaction
    _check(lib.dgb_assemble_nonlinear_host(C.byref(mesh.view), C.byref(ref.view), coef.ctypes.data,
                                           coef.shape[0], C.byref(r), device, h.ctypes.data,
                                           C.byref(b)))
    return h, (row_ptr, col, val)


def _stream_handle(device: int, stream=None) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def solve_options(tolerance_scale: float | None = None, max_iterations: int | None = None,
                  restart: int | None = None, preconditioner: int | None = None) -> "capi.SolveOptions":
    o = capi.SolveOptions()
    capi.load().dgb_solve_options_default(C.byref(o))
    if preconditioner is not None:
        o.preconditioner = preconditioner
    if tolerance_scale is not None:
        o.tolerance_scale = tolerance_scale
    if max_iterations is not None:
        o.max_iterations = max_iterations
    if restart is not None:
        o.restart = restart
    return o


def solve(system: BsrSystem, b, x=None, options=None, device: int = 0, stream=None):
    """`direct_solve(stiffness(), b, &info)` (sparse.cpp:154-217) on the device: block-Jacobi
    GMRES(m) under the reference's accuracy contract.  b, x: device tensors [n] (x = initial
    guess, zeros by default).  Returns (x, info dict); raises Error(SingularMatrix /
    SolveAccuracy / DimensionMismatch) like the reference."""
    import torch
    lib = capi.load()
    n = (system.row_ptr.shape[0] - 1) * system.block_dim
    if b.numel() != n:
        raise Error(capi.STATUS_NAMES.index("DimensionMismatch"), "right-hand side size mismatch", -1)
    if x is None:
        x = torch.zeros(n, dtype=torch.float64, device=b.device)
    info = capi.SolveInfo()
    bs = system.struct()
    _check(lib.dgb_solve(C.byref(bs), b.data_ptr(), x.data_ptr(),
                         C.byref(options) if options is not None else None, C.byref(info),
                         C.c_void_p(_stream_handle(device, stream))))
    return x, {"defect_norm2": info.defect_norm2, "defect_norm_inf": info.defect_norm_inf,
               "bound": info.bound, "iterations": info.iterations, "restarts": info.restarts}


def newton_config(max_iterations: int = 50, residual_tolerance: float = 1e-10,
                  step_tolerance: float = 1e-12, legacy_check: float | None = None):
    c = capi.NewtonConfig()
    c.max_iterations, c.residual_tolerance, c.step_tolerance = max_iterations, residual_tolerance, step_tolerance
    c.use_legacy_check = int(legacy_check is not None)
    c.legacy_check = legacy_check if legacy_check is not None else 0.0
    return c


def newton_solve(plan: Plan, dmesh: DeviceMesh, system: BsrSystem, reaction: int, config=None,
                 initial_guess=None, options=None, stream=None):
    """`newton_solve(system, mesh, ref, reaction, config, initial_guess)`
    (nonlinear.cpp:109-176) on the device.  Returns (coef tensor, report dict)."""
    import torch
    lib = capi.load()
    n = dmesh.n_elements * plan.n_local
    cfg = config if config is not None else newton_config()
    if initial_guess is None:
        coef = torch.zeros(n, dtype=torch.float64, device=system.val.device)
    else:
        coef = initial_guess.clone()
    hist = np.zeros(max(cfg.max_iterations, 1))
    rep = capi.NewtonReport()
    rep.residual_history = hist.ctypes.data
    r = capi.Reaction()
    r.kind = reaction
    bs = system.struct()
    _check(lib.dgb_newton_solve(plan._h, C.byref(dmesh.view), C.byref(bs),
                                system.rhs.data_ptr(), C.byref(r), C.byref(cfg),
                                C.byref(options) if options is not None else None,
                                coef.data_ptr(), C.byref(rep),
                                C.c_void_p(_stream_handle(plan.device, stream))))
    return coef, {"iterations": rep.iterations, "converged": bool(rep.converged),
                  "final_residual": rep.final_residual,
                  "residual_history": hist[:rep.iterations].tolist(),
                  "linear_iterations": rep.linear_iterations}


# ------------------------------------------------------------------------------ postprocess
def l2_error(coef, dmesh: DeviceMesh, ref: ReferenceElement, exact, device: int = 0, stream=None):
    """`l2_error(coef, mesh, ref, exact)` (postprocess.cpp:14-50) on the device: coef a device
    tensor [E * nl], exact a ScalarField descriptor (capi.ScalarField, e.g. problems.function).
    Returns (error, h_max)."""
    lib = capi.load()
    sharp = ReferenceElement(ref.degree, lib.dgb_l2_quad_order(ref.degree, ref.quad_order))
    plan = Plan(sharp.view, device)
    out = (C.c_double * 2)()
    _check(lib.dgb_l2_error(plan._h, C.byref(dmesh.view), coef.data_ptr(), coef.numel(),
                            C.byref(exact), out, C.c_void_p(_stream_handle(device, stream))))
    return out[0], out[1]


def project(dmesh: DeviceMesh, ref: ReferenceElement, f, device: int = 0, stream=None):
    """`project(mesh, ref, f)` (postprocess.cpp:56-81): device tensor [E * nl]."""
    import torch
    lib = capi.load()
    plan = Plan(ref.view, device)
    coef = torch.empty(dmesh.n_elements * ref.n_local, dtype=torch.float64,
                       device=torch.device("cuda", device))
    _check(lib.dgb_project(plan._h, C.byref(dmesh.view), C.byref(f), coef.data_ptr(),
                           C.c_void_p(_stream_handle(device, stream))))
    return coef


def eval_solution(coef, ref: ReferenceElement, elements, xhat, yhat, device: int = 0, stream=None):
    """`eval_solution(coef, ref, element, xhat, yhat)` (postprocess.cpp:83-93) for a batch of
    points (device tensors); returns a device tensor of values."""
    import torch
    lib = capi.load()
    n = elements.numel()
    out = torch.empty(n, dtype=torch.float64, device=coef.device)
    _check(lib.dgb_eval_solution(coef.data_ptr(), ref.degree, coef.numel() // ref.n_local, n,
                                 elements.data_ptr(), xhat.data_ptr(), yhat.data_ptr(),
                                 out.data_ptr(), C.c_void_p(_stream_handle(device, stream))))
    return out


# ------------------------------------------------------------------------------ device mesh build
class DeviceBuiltMesh:
    """A mesh built in HBM by dgb_device_mesh_build / dgb_device_mesh_refine (build_mesh and
    uniform_refine, mesh.cpp:51-187).  Usable wherever a DeviceMesh is (`.view`)."""

    def __init__(self, handle, device: int = 0):
        self._lib = capi.load()
        self._h = handle
        self.device = device
        v = MeshArrays()
        _check(self._lib.dgb_device_mesh_view(handle, C.byref(v)))
        self.view = v
        self.n_nodes, self.n_elements, self.n_edges = v.n_nodes, v.n_elements, v.n_edges
        self.n_interior_edges = v.n_interior_edges

    def refine(self, stream=None) -> "DeviceBuiltMesh":
        h = C.c_void_p()
        _check(self._lib.dgb_device_mesh_refine(self._h, C.byref(h),
                                                C.c_void_p(_stream_handle(self.device, stream))))
        return DeviceBuiltMesh(h, self.device)

    def arrays(self) -> dict:
        """Host copies of the mesh arrays (the layout of Mesh.arrays())."""
        v = self.view
        out = {"nodes": np.zeros((v.n_nodes, 2)), "elements": np.zeros((v.n_elements, 3), np.int32),
               "edges": np.zeros((v.n_edges, 2), np.int32), "edge_kind": np.zeros(v.n_edges, np.uint8),
               "edge_elements": np.zeros((v.n_edges, 2), np.int32),
               "element_edges": np.zeros((v.n_elements, 3), np.int32)}
        _check(self._lib.dgb_device_mesh_copy_to_host(
            self._h, *(out[k].ctypes.data for k in ("nodes", "elements", "edges", "edge_kind",
                                                     "edge_elements", "element_edges"))))
        return out

    def __del__(self):
        try:
            self._lib.dgb_device_mesh_free(self._h)
        except Exception:
            pass


def device_build_mesh(nodes, elements, dirichlet, neumann, device: int = 0,
                      stream=None) -> DeviceBuiltMesh:
    """build_mesh(nodes, elements, dirichlet, neumann) (mesh.cpp:51-151) on the device; host
    numpy or device torch inputs.  Raises Error like the reference."""
    lib = capi.load()

    def ptr(a, dtype):
        if hasattr(a, "data_ptr"):
            return a.data_ptr(), a
        arr = np.ascontiguousarray(a, dtype=dtype)
        return arr.ctypes.data, arr
    pn, kn = ptr(nodes, np.float64)
    pe, ke = ptr(elements, np.int32)
    pd, kd = ptr(dirichlet, np.int32)
    pm, km = ptr(neumann, np.int32)
    count = (lambda a, w: (a.numel() if hasattr(a, "numel") else np.asarray(a).size) // w)
    h = C.c_void_p()
    _check(lib.dgb_device_mesh_build(pn, count(nodes, 2), pe, count(elements, 3), pd,
                                     count(dirichlet, 2), pm, count(neumann, 2), device, C.byref(h),
                                     C.c_void_p(_stream_handle(device, stream))))
    del kn, ke, kd, km
    return DeviceBuiltMesh(h, device)
