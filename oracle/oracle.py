"""TEST INFRASTRUCTURE -- ctypes wrappers of the two CPU checkers.

* `RefLib`   : oracle/_ref/libdgref.so, the UNMODIFIED reference (built from /root/reference by
               oracle/Makefile; the prebuilt .so travels to the GPU box).
* `OracleLib`: oracle/libdgoracle.so, the plain-C restatement dg_oracle.c.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module, and only as the checker (never on the product path).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1502_02941_b200 import capi
from paper_1502_02941_b200.capi import MeshArrays, Params, Problem, ReferenceTables

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libdgref.so")
ORACLE_SO = os.path.join(HERE, "libdgoracle.so")
REFERENCE_SRC = "/root/reference/proj"


def build(ref: bool | None = None) -> None:
    """Builds the restatement, and the reference when its sources are present."""
    subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)
    if ref is None:
        ref = os.path.isdir(os.path.join(REFERENCE_SRC, "src"))
    if ref:
        subprocess.run(["make", "-j8", "-C", HERE, "ref"], check=True, capture_output=True)


def _ptr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data


def mesh_arrays_from_numpy(d: dict) -> MeshArrays:
    """A MeshArrays over numpy arrays (the dict keeps them alive)."""
    m = MeshArrays()
    m.n_nodes = d["nodes"].shape[0]
    m.n_elements = d["elements"].shape[0]
    m.n_edges = d["edges"].shape[0]
    m.n_interior_edges = int((d["edge_kind"] == capi.EDGE_INTERIOR).sum())
    for k in ("nodes", "elements", "edges", "edge_kind", "edge_elements", "element_edges"):
        setattr(m, k, d[k].ctypes.data)
    return m


def mesh_numpy_from_arrays(m: MeshArrays) -> dict:
    """Copies a MeshArrays (host pointers) into numpy arrays."""
    def arr(ptr, n, ct, shape):
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).copy().reshape(shape)
    return {
        "nodes": arr(m.nodes, 2 * m.n_nodes, C.c_double, (m.n_nodes, 2)),
        "elements": arr(m.elements, 3 * m.n_elements, C.c_int32, (m.n_elements, 3)),
        "edges": arr(m.edges, 2 * m.n_edges, C.c_int32, (m.n_edges, 2)),
        "edge_kind": arr(m.edge_kind, m.n_edges, C.c_uint8, (m.n_edges,)),
        "edge_elements": arr(m.edge_elements, 2 * m.n_edges, C.c_int32, (m.n_edges, 2)),
        "element_edges": arr(m.element_edges, 3 * m.n_elements, C.c_int32, (m.n_elements, 3)),
    }


def tables_numpy_from_view(t: ReferenceTables) -> dict:
    nl, nq, ne = t.n_local, t.nq_vol, t.nq_edge

    def arr(ptr, n):
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(n,)).copy()
    return {
        "degree": t.degree, "n_local": nl, "nq_vol": nq, "nq_edge": ne,
        "vol_x": arr(t.vol_x, nq), "vol_y": arr(t.vol_y, nq), "vol_w": arr(t.vol_w, nq),
        "edge_t": arr(t.edge_t, ne), "edge_w": arr(t.edge_w, ne),
        "phi": arr(t.phi, nq * nl), "dphi": arr(t.dphi, nq * nl * 2),
        "edge_phi": arr(t.edge_phi, 6 * ne * nl), "edge_dphi": arr(t.edge_dphi, 6 * ne * nl * 2),
    }


def tables_view_from_numpy(d: dict) -> ReferenceTables:
    t = ReferenceTables()
    t.degree, t.n_local, t.nq_vol, t.nq_edge = d["degree"], d["n_local"], d["nq_vol"], d["nq_edge"]
    for k in ("vol_x", "vol_y", "vol_w", "edge_t", "edge_w", "phi", "dphi", "edge_phi",
              "edge_dphi"):
        setattr(t, k, d[k].ctypes.data)
    return t


class ReferenceError_(RuntimeError):
    def __init__(self, status: int, message: str, detail: int):
        super().__init__(message)
        self.status = status
        self.code = capi.STATUS_NAMES[status] if 0 <= status < len(capi.STATUS_NAMES) else str(status)
        self.detail = detail


class RefLib:
    """The compiled reference behind ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = C.CDLL(path)
        vp = C.c_void_p
        P = C.POINTER
        sig = {
            "dgref_last_error": (C.c_char_p, []),
            "dgref_last_detail": (C.c_long, []),
            "dgref_build_mesh": (C.c_int, [vp, C.c_int, vp, C.c_int, vp, C.c_int, vp, C.c_int, P(vp)]),
            "dgref_unit_square_refined": (C.c_int, [C.c_int, C.c_int, P(vp)]),
            "dgref_mesh_view": (C.c_int, [vp, P(MeshArrays)]),
            "dgref_mesh_free": (None, [vp]),
            "dgref_reference": (C.c_int, [C.c_int, C.c_int, P(vp)]),
            "dgref_reference_view": (C.c_int, [vp, P(ReferenceTables)]),
            "dgref_reference_free": (None, [vp]),
            "dgref_set_parameters": (C.c_int, [C.c_int, C.c_int, P(Params)]),
            "dgref_assemble": (C.c_int, [vp, vp, P(Problem), P(Params), C.c_int, C.c_int,
                                         P(C.c_double), P(vp)]),
            "dgref_assemble_convection": (C.c_int, [vp, vp, P(Problem), C.c_int]),
            "dgref_system_nnz": (C.c_int, [vp, C.c_int, P(C.c_longlong), P(C.c_int)]),
            "dgref_system_copy": (C.c_int, [vp, C.c_int, vp, vp, vp]),
            "dgref_system_rhs": (C.c_int, [vp, vp]),
            "dgref_matvec": (C.c_int, [vp, vp, vp]),
            "dgref_system_free": (None, [vp]),
            "dgref_element_geometry": (C.c_int, [vp, C.c_int, vp]),
            "dgref_edge_geometry": (C.c_int, [vp, C.c_int, vp]),
            "dgref_assemble_nonlinear": (C.c_int, [vp, vp, vp, C.c_longlong, C.c_int, C.c_int,
                                                   vp, vp, vp, vp, P(C.c_double)]),
            "dgref_l2_error": (C.c_int, [vp, vp, vp, C.c_longlong, vp, vp]),
            "dgref_project": (C.c_int, [vp, vp, vp, vp]),
            "dgref_eval_solution": (C.c_int, [vp, C.c_longlong, vp, C.c_longlong, vp, vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        self.lib = lib

    def _check(self, status: int) -> None:
        if status != 0:
            raise ReferenceError_(status, self.lib.dgref_last_error().decode(),
                                  int(self.lib.dgref_last_detail()))

    # -- mesh ---------------------------------------------------------------------------
    def build_mesh(self, nodes, elements, dirichlet, neumann) -> "RefMesh":
        nodes = np.ascontiguousarray(nodes, dtype=np.float64)
        elements = np.ascontiguousarray(elements, dtype=np.int32)
        dirichlet = np.ascontiguousarray(dirichlet, dtype=np.int32).reshape(-1, 2)
        neumann = np.ascontiguousarray(neumann, dtype=np.int32).reshape(-1, 2)
        h = C.c_void_p()
        self._check(self.lib.dgref_build_mesh(
            _ptr(nodes), nodes.shape[0], _ptr(elements), elements.shape[0],
            _ptr(dirichlet), dirichlet.shape[0], _ptr(neumann), neumann.shape[0], C.byref(h)))
        return RefMesh(self, h)

    def unit_square_refined(self, levels: int, neumann_sides: int = 0) -> "RefMesh":
        h = C.c_void_p()
        self._check(self.lib.dgref_unit_square_refined(levels, neumann_sides, C.byref(h)))
        return RefMesh(self, h)

    # -- reference element ----------------------------------------------------------------
    def reference(self, degree: int, quad_order: int = 0) -> "RefElement":
        h = C.c_void_p()
        self._check(self.lib.dgref_reference(degree, quad_order, C.byref(h)))
        return RefElement(self, h)

    def set_parameters(self, method: int, degree: int) -> Params:
        p = Params()
        self._check(self.lib.dgref_set_parameters(method, degree, C.byref(p)))
        return p

    # -- assembly -------------------------------------------------------------------------
    def assemble(self, mesh: "RefMesh", ref: "RefElement", problem: Problem, params: Params,
                 threads: int = 0, clip_sides: int = 0) -> "RefSystem":
        h = C.c_void_p()
        secs = (C.c_double * 2)()
        self._check(self.lib.dgref_assemble(mesh.h, ref.h, C.byref(problem), C.byref(params),
                                            threads, clip_sides, secs, C.byref(h)))
        return RefSystem(self, h, ref.tables["n_local"], (secs[0], secs[1]))

    def assemble_convection(self, mesh, ref, problem, threads: int = 0) -> None:
        self._check(self.lib.dgref_assemble_convection(mesh.h, ref.h, C.byref(problem), threads))

    def l2_error(self, mesh: "RefMesh", ref: "RefElement", coef: np.ndarray, exact) -> tuple:
        coef = np.ascontiguousarray(coef, dtype=np.float64)
        out = np.zeros(2)
        self._check(self.lib.dgref_l2_error(mesh.h, ref.h, _ptr(coef), coef.shape[0],
                                            C.byref(exact), _ptr(out)))
        return float(out[0]), float(out[1])

    def project(self, mesh: "RefMesh", ref: "RefElement", f, n_elements: int) -> np.ndarray:
        out = np.zeros(n_elements * ref.tables["n_local"])
        self._check(self.lib.dgref_project(mesh.h, ref.h, C.byref(f), _ptr(out)))
        return out

    def eval_solution(self, coef, ref: "RefElement", elements, xh, yh) -> np.ndarray:
        coef = np.ascontiguousarray(coef, dtype=np.float64)
        elements = np.ascontiguousarray(elements, dtype=np.int32)
        xh = np.ascontiguousarray(xh, dtype=np.float64)
        yh = np.ascontiguousarray(yh, dtype=np.float64)
        out = np.zeros(elements.shape[0])
        self._check(self.lib.dgref_eval_solution(_ptr(coef), coef.shape[0], ref.h, elements.shape[0],
                                                 _ptr(elements), _ptr(xh), _ptr(yh), _ptr(out)))
        return out

    def assemble_nonlinear(self, mesh: "RefMesh", ref: "RefElement", coef: np.ndarray, kind: int,
                           threads: int = 0):
        """dgfem::assemble_nonlinear: returns (h, (row_offsets, cols, vals), seconds)."""
        coef = np.ascontiguousarray(coef, dtype=np.float64)
        nl = ref.tables["n_local"]
        n = coef.shape[0]
        ne = n // nl if nl else 0
        h = np.zeros(n)
        ro = np.zeros(n + 1, np.int32)
        cols = np.zeros(ne * nl * nl, np.int32)
        vals = np.zeros(ne * nl * nl)
        secs = (C.c_double * 1)()
        self._check(self.lib.dgref_assemble_nonlinear(mesh.h, ref.h, _ptr(coef), n, kind, threads,
                                                      _ptr(h), _ptr(ro), _ptr(cols), _ptr(vals),
                                                      secs))
        return h, (ro, cols, vals), secs[0]


class RefMesh:
    def __init__(self, lib: RefLib, h: C.c_void_p):
        self.lib, self.h = lib, h
        v = MeshArrays()
        lib.lib.dgref_mesh_view(h, C.byref(v))
        self.view = v
        self.arrays = mesh_numpy_from_arrays(v)

    def element_geometry(self, e: int) -> np.ndarray:
        out = np.zeros(13)
        self.lib._check(self.lib.lib.dgref_element_geometry(self.h, e, _ptr(out)))
        return out

    def edge_geometry(self, edge: int) -> np.ndarray:
        out = np.zeros(6)
        self.lib._check(self.lib.lib.dgref_edge_geometry(self.h, edge, _ptr(out)))
        return out

    def __del__(self):
        try:
            self.lib.lib.dgref_mesh_free(self.h)
        except Exception:
            pass


class RefElement:
    def __init__(self, lib: RefLib, h: C.c_void_p):
        self.lib, self.h = lib, h
        v = ReferenceTables()
        lib.lib.dgref_reference_view(h, C.byref(v))
        self.tables = tables_numpy_from_view(v)

    def __del__(self):
        try:
            self.lib.lib.dgref_reference_free(self.h)
        except Exception:
            pass


class RefSystem:
    """assemble_all's DgSystem + stiffness(); matrices are returned as CSR numpy triples."""

    def __init__(self, lib: RefLib, h: C.c_void_p, nl: int, seconds):
        self.lib, self.h, self.nl, self.seconds = lib, h, nl, seconds

    def csr(self, which: int = 0):
        nnz, n = C.c_longlong(), C.c_int()
        self.lib.lib.dgref_system_nnz(self.h, which, C.byref(nnz), C.byref(n))
        rp = np.zeros(n.value + 1, np.int32)
        ci = np.zeros(nnz.value, np.int32)
        va = np.zeros(nnz.value, np.float64)
        self.lib.lib.dgref_system_copy(self.h, which, _ptr(rp), _ptr(ci), _ptr(va))
        return rp, ci, va

    def rhs(self) -> np.ndarray:
        _, n = C.c_longlong(), C.c_int()
        self.lib.lib.dgref_system_nnz(self.h, 0, C.byref(_), C.byref(n))
        F = np.zeros(n.value)
        self.lib.lib.dgref_system_rhs(self.h, _ptr(F))
        return F

    def matvec(self, x: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """The reference's own matvec (sparse.cpp:116-129) of stiffness() with x."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        nnz, n = C.c_longlong(), C.c_int()
        self.lib.lib.dgref_system_nnz(self.h, 0, C.byref(nnz), C.byref(n))
        y = np.zeros(n.value) if out is None else out
        self.lib._check(self.lib.lib.dgref_matvec(self.h, _ptr(x), _ptr(y)))
        return y

    def __del__(self):
        try:
            self.lib.lib.dgref_system_free(self.h)
        except Exception:
            pass


class OracleLib:
    """The plain-C restatement (dg_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        lib = C.CDLL(path)
        vp = C.c_void_p
        lib.dgo_count_blocks.restype = C.c_int64
        lib.dgo_count_blocks.argtypes = [C.POINTER(MeshArrays), vp, C.c_int32]
        lib.dgo_assemble.restype = C.c_int
        lib.dgo_assemble.argtypes = [C.POINTER(MeshArrays), C.POINTER(ReferenceTables),
                                     C.POINTER(Problem), C.POINTER(Params), vp, C.c_int32,
                                     C.c_int32, vp, vp, vp, vp, C.POINTER(C.c_longlong)]
        lib.dgo_spmv.restype = None
        lib.dgo_spmv.argtypes = [vp, vp, vp, C.c_int32, C.c_int32, vp, vp, C.c_int32]
        lib.dgo_assemble_nonlinear.restype = C.c_int
        lib.dgo_assemble_nonlinear.argtypes = [C.POINTER(MeshArrays), C.POINTER(ReferenceTables),
                                               vp, C.c_int64, C.c_int32, vp, C.c_int32, C.c_int32,
                                               vp, vp]
        lib.dgo_l2_error.restype = C.c_int
        lib.dgo_l2_error.argtypes = [C.POINTER(MeshArrays), C.POINTER(ReferenceTables), vp, C.c_int64,
                                     vp, vp]
        lib.dgo_project.restype = C.c_int
        lib.dgo_project.argtypes = [C.POINTER(MeshArrays), C.POINTER(ReferenceTables), vp, vp]
        lib.dgo_eval_solution.restype = C.c_int
        lib.dgo_eval_solution.argtypes = [vp, C.c_int32, C.c_int64, vp, vp, vp, vp]
        self.lib = lib

    def l2_error(self, mesh: dict, sharp_tables: dict, coef, exact) -> tuple:
        """postprocess.cpp:14-50 with the sharper rule's tables (see dgb_l2_quad_order)."""
        m = mesh_arrays_from_numpy(mesh)
        t = tables_view_from_numpy(sharp_tables)
        coef = np.ascontiguousarray(coef, dtype=np.float64)
        out = np.zeros(2)
        st = self.lib.dgo_l2_error(C.byref(m), C.byref(t), _ptr(coef), coef.shape[0],
                                   C.addressof(exact), _ptr(out))
        if st != 0:
            raise ReferenceError_(st, capi.STATUS_NAMES[st], -1)
        return float(out[0]), float(out[1])

    def project(self, mesh: dict, tables: dict, f) -> np.ndarray:
        m = mesh_arrays_from_numpy(mesh)
        t = tables_view_from_numpy(tables)
        out = np.zeros(mesh["elements"].shape[0] * tables["n_local"])
        self.lib.dgo_project(C.byref(m), C.byref(t), C.addressof(f), _ptr(out))
        return out

    def eval_solution(self, coef, degree: int, elements, xh, yh) -> np.ndarray:
        coef = np.ascontiguousarray(coef, dtype=np.float64)
        elements = np.ascontiguousarray(elements, dtype=np.int32)
        xh = np.ascontiguousarray(xh, dtype=np.float64)
        yh = np.ascontiguousarray(yh, dtype=np.float64)
        out = np.zeros(elements.shape[0])
        self.lib.dgo_eval_solution(_ptr(coef), degree, elements.shape[0], _ptr(elements),
                                   _ptr(xh), _ptr(yh), _ptr(out))
        return out

    def assemble_nonlinear(self, mesh: dict, tables: dict, coef: np.ndarray, kind: int,
                           rows: np.ndarray | None = None, threads: int = 0):
        """H and the HJ blocks of elements `rows` (default all): (h [n, nl], hj [n, nl, nl])."""
        m = mesh_arrays_from_numpy(mesh)
        t = tables_view_from_numpy(tables)
        nl = tables["n_local"]
        coef = np.ascontiguousarray(coef, dtype=np.float64)
        if threads <= 0:
            threads = os.cpu_count() or 1
        if rows is not None:
            rows = np.ascontiguousarray(rows, dtype=np.int32)
        n = mesh["elements"].shape[0] if rows is None else rows.shape[0]
        h = np.zeros((n, nl))
        hj = np.zeros((n, nl, nl))
        st = self.lib.dgo_assemble_nonlinear(C.byref(m), C.byref(t), _ptr(coef), coef.shape[0],
                                             kind, _ptr(rows), n, threads, _ptr(h), _ptr(hj))
        if st != 0:
            raise ReferenceError_(st, capi.STATUS_NAMES[st], -1)
        return h, hj

    def assemble(self, mesh: dict, tables: dict, problem: Problem, params: Params,
                 rows: np.ndarray | None = None, threads: int = 0):
        """Block rows `rows` (default all) of K and F: returns (row_ptr, col, val, rhs) with
        val shaped [nblocks, nl, nl] and rhs [n_rows, nl]; raises ReferenceError_."""
        m = mesh_arrays_from_numpy(mesh)
        t = tables_view_from_numpy(tables)
        nl = tables["n_local"]
        if threads <= 0:
            threads = os.cpu_count() or 1
        if rows is not None:
            rows = np.ascontiguousarray(rows, dtype=np.int32)
        n = mesh["elements"].shape[0] if rows is None else rows.shape[0]
        nb = self.lib.dgo_count_blocks(C.byref(m), _ptr(rows), n)
        row_ptr = np.zeros(n + 1, np.int32)
        col = np.zeros(nb, np.int32)
        val = np.zeros((nb, nl, nl))
        rhs = np.zeros((n, nl))
        detail = C.c_longlong(-1)
        st = self.lib.dgo_assemble(C.byref(m), C.byref(t), C.byref(problem), C.byref(params),
                                   _ptr(rows), n, threads, _ptr(row_ptr), _ptr(col), _ptr(val),
                                   _ptr(rhs), C.byref(detail))
        if st != 0:
            raise ReferenceError_(st, capi.STATUS_NAMES[st], detail.value)
        return row_ptr, col, val, rhs

    def spmv(self, row_ptr, col, val, x, threads: int = 0) -> np.ndarray:
        nl = val.shape[1]
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros((row_ptr.shape[0] - 1) * nl)  # rows of the (possibly sharded) BSR
        self.lib.dgo_spmv(_ptr(row_ptr), _ptr(col), _ptr(val), nl, row_ptr.shape[0] - 1,
                          _ptr(x), _ptr(y), threads if threads > 0 else (os.cpu_count() or 1))
        return y


def bsr_to_csr(row_ptr, col, val):
    """Expands a sorted BSR (val [nb, nl, nl]) into the reference's CSR (sorted columns)."""
    nl = val.shape[1]
    n_rows = row_ptr.shape[0] - 1
    nb_row = np.diff(row_ptr)
    # entries of block row e, row i: all blocks of e in order, each contributing nl columns
    rp = np.zeros(n_rows * nl + 1, np.int64)
    rp[1:] = np.repeat(nb_row * nl, nl).cumsum()
    cols = np.empty(rp[-1], np.int32)
    vals = np.empty(rp[-1])
    for e in range(n_rows):
        b0, b1 = row_ptr[e], row_ptr[e + 1]
        c = (col[b0:b1, None] * nl + np.arange(nl)[None, :]).reshape(-1)
        for i in range(nl):
            s = rp[e * nl + i]
            cols[s:s + c.size] = c
            vals[s:s + c.size] = val[b0:b1, i, :].reshape(-1)
    return rp, cols, vals
