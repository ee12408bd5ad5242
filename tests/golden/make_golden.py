"""Generates the committed golden fixtures from the UNMODIFIED reference library.

Run in a container where /root/reference exists (it is absent on the GPU box):

    make -C oracle ref && python tests/golden/make_golden.py

Everything here comes out of oracle/_ref/libdgref.so, i.e. the reference's own build_mesh,
ReferenceElement, assemble_all + stiffness() and error reporting, called through
oracle/ref_shim.cpp.  The reference ships no golden data files, so these
fixtures are what pins the plain-C restatement (oracle/dg_oracle.c) and the host-side
mesh / table builders when the reference itself is not available.

Outputs (numpy .npz, a few MB in total):
  tables.npz   ReferenceElement tables, degrees 1..4, quad_order 0 and 2k+1
  meshes.npz   build_mesh inputs and outputs, plus the reference's error codes/details
  systems.npz  assembled K (CSR) and F for small meshes: every BASELINE config's
               coefficients, the registry problems the reference tests use, all methods
  nonlinear.npz  assemble_nonlinear's H and HJ (CSR), degrees 1..4, every reaction kind,
               seeded coefficients; plus the coefficient-length error
  postprocess.npz  l2_error, project and eval_solution, degrees 1..4
  refine.npz   unit_square_mesh + uniform_refine, levels 0 and 4

    python tests/golden/make_golden.py [tables meshes systems nonlinear]   (default: all)
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import ReferenceError_, RefLib  # noqa: E402
from paper_1502_02941_b200 import capi, dgfem, problems  # noqa: E402

METHODS = {"sipg": capi.SIPG, "nipg": capi.NIPG, "iipg": capi.IIPG}


def tables(ref: RefLib) -> dict:
    out = {}
    for k in (1, 2, 3, 4):
        for qo in (0, 2 * k + 1):
            t = ref.reference(k, qo).tables
            for name, v in t.items():
                out[f"k{k}_q{qo}_{name}"] = np.asarray(v)
    return out


def mesh_cases():
    """(name, raw mesh dict) from the repo's generators, plus the reference tests' meshes."""
    cases = []
    for n, jit, perm, sides in [(3, 0.0, False, 0), (5, 0.2, True, 2 | 8), (6, 0.0, True, 0),
                                (4, 0.2, False, 1 | 4)]:
        m = dgfem.unit_square_mesh(n, jit, 17 + n, perm, 29 + n, sides)
        cases.append((f"square{n}_j{int(jit * 10)}_p{int(perm)}_s{sides}", m.raw()))
    # test_assembly.cpp:44-48 two_element_square
    cases.append(("two_element", {
        "nodes": np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float),
        "elements": np.array([[0, 1, 2], [0, 2, 3]], np.int32),
        "dirichlet": np.array([[0, 1], [1, 2], [2, 3], [0, 3]], np.int32),
        "neumann": np.zeros((0, 2), np.int32)}))
    # a clockwise element (reoriented by build_mesh, mesh.cpp:70-72)
    cases.append(("clockwise", {
        "nodes": np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float),
        "elements": np.array([[0, 2, 1], [0, 2, 3]], np.int32),
        "dirichlet": np.array([[0, 1], [1, 2], [2, 3], [0, 3]], np.int32),
        "neumann": np.zeros((0, 2), np.int32)}))
    return cases


ERROR_CASES = {
    # name: (nodes, elements, dirichlet, neumann)
    "bad_node_index": ([[0, 0], [1, 0], [0, 1]], [[0, 1, 3]], [[0, 1], [1, 2], [0, 2]], []),
    "degenerate": ([[0, 0], [1, 0], [2, 0], [0, 1]], [[0, 3, 1], [0, 1, 2]], [], []),
    "non_manifold": ([[0, 0], [1, 0], [0, 1], [0, -1], [1, 1]],
                     [[0, 1, 2], [0, 3, 1], [0, 1, 4]], [], []),
    "unknown_pair": ([[0, 0], [1, 0], [0, 1]], [[0, 1, 2]], [[0, 1], [1, 2], [0, 2], [0, 5]], []),
    "interior_pair": ([[0, 0], [1, 0], [1, 1], [0, 1]], [[0, 1, 2], [0, 2, 3]],
                      [[0, 1], [1, 2], [2, 3], [0, 3], [0, 2]], []),
    "tagged_twice": ([[0, 0], [1, 0], [0, 1]], [[0, 1, 2]], [[0, 1], [1, 2], [0, 2]], [[1, 0]]),
    "untagged": ([[0, 0], [1, 0], [0, 1]], [[0, 1, 2]], [[0, 1], [1, 2]], []),
}


def meshes(ref: RefLib) -> dict:
    out = {}
    for name, raw in mesh_cases():
        m = ref.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
        for k, v in raw.items():
            out[f"{name}/in_{k}"] = np.asarray(v)
        for k, v in m.arrays.items():
            out[f"{name}/out_{k}"] = v
    for name, (nodes, el, d, nm) in ERROR_CASES.items():
        try:
            ref.build_mesh(np.array(nodes, float), np.array(el, np.int32),
                           np.array(d, np.int32).reshape(-1, 2), np.array(nm, np.int32).reshape(-1, 2))
            status, detail = 0, -1
        except ReferenceError_ as e:
            status, detail = e.status, e.detail
        out[f"err_{name}/nodes"] = np.array(nodes, float)
        out[f"err_{name}/elements"] = np.array(el, np.int32)
        out[f"err_{name}/dirichlet"] = np.array(d, np.int32).reshape(-1, 2)
        out[f"err_{name}/neumann"] = np.array(nm, np.int32).reshape(-1, 2)
        out[f"err_{name}/status"] = np.array(status)
        out[f"err_{name}/detail"] = np.array(detail)
    return out


def system_cases():
    """(name, mesh raw dict, degree, quad_order, ProblemSpec, params, clip_sides)."""
    cases = []
    for idx in (1, 2, 3, 4, 5):
        cfg = problems.CONFIGS[idx]
        n = 6
        m = dgfem.unit_square_mesh(n, cfg.jitter, problems.SEED_JITTER, cfg.permute,
                                   problems.SEED_PERMUTE, cfg.neumann_sides)
        spec = problems.config_problem(idx, m.n_elements)
        for meth in cfg.methods:
            p = dgfem.config_parameters(cfg, meth)
            clip = cfg.neumann_sides if cfg.neumann_inflow == capi.INFLOW_DROP else 0
            cases.append((f"config{idx}_{['sipg', 'nipg', 'iipg'][meth]}", m.raw(), cfg.degree,
                          cfg.quad_order, spec, p, clip))
    reg = [("smooth-sine", 2, "sipg"), ("smooth-sine", 3, "nipg"), ("smooth-sine-mixed", 1, "iipg"),
           ("poly-exact", 1, "sipg"), ("paper-boundary-layer-linear", 2, "sipg"),
           ("pure-advection-patch", 4, "iipg")]
    for name, k, meth in reg:
        spec = problems.registry_get(name)
        m = dgfem.unit_square_mesh(4, 0.15, 3, True, 4, spec.neumann_sides)
        p = dgfem.set_parameters(METHODS[meth], k)
        cases.append((f"{name}_k{k}_{meth}", m.raw(), k, 0, spec, p, 0))
    # two_element_square with constant wind (2, 1) (test_assembly.cpp:302-326)
    spec = problems.registry_get("poly-exact")
    spec.c.advection = problems.vec_constant(2.0, 1.0)
    raw = dict(mesh_cases())["two_element"]
    for k in (1, 2):
        cases.append((f"two_element_k{k}", raw, k, 0, spec, dgfem.set_parameters(capi.SIPG, k), 0))
    return cases


def systems(ref: RefLib) -> dict:
    out = {}
    for name, raw, k, qo, spec, p, clip in system_cases():
        mesh = ref.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
        r = ref.reference(k, qo)
        s = ref.assemble(mesh, r, spec.c, p, threads=1, clip_sides=clip)
        rp, ci, va = s.csr(0)
        out[f"{name}/row_offsets"] = rp
        out[f"{name}/cols"] = ci
        out[f"{name}/vals"] = va
        out[f"{name}/F"] = s.rhs()
        out[f"{name}/degree"] = np.array(k)
        out[f"{name}/quad_order"] = np.array(qo)
        out[f"{name}/params"] = np.array([p.method, p.degree, p.kappa, p.sigma_interior,
                                          p.sigma_boundary, p.neumann_inflow], float)
        for kk, v in raw.items():
            out[f"{name}/in_{kk}"] = np.asarray(v)
        for field, arr in spec.per_element.items():
            out[f"{name}/per_element_{field}"] = arr
    # InflowOnNeumann: smooth-sine (b = (1, 2)) on the all-Neumann unit square
    # (test_assembly.cpp:371-381, test_parallel_consistency.cpp:152-182)
    m = dgfem.unit_square_mesh(4, 0.0, 0, False, 0, 15)
    raw = m.raw()
    rmesh = ref.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
    try:
        ref.assemble_convection(rmesh, ref.reference(1, 0), problems.registry_get("smooth-sine").c)
        detail = -1
    except ReferenceError_ as e:
        assert e.code == "InflowOnNeumann", e.code
        detail = e.detail
    for kk, v in raw.items():
        out[f"inflow_on_neumann/in_{kk}"] = np.asarray(v)
    out["inflow_on_neumann/detail"] = np.array(detail)
    return out


REACTIONS = {"zero": capi.REACTION_ZERO, "linear": capi.REACTION_LINEAR,
             "square": capi.REACTION_SQUARE, "cubic": capi.REACTION_CUBIC}


def nonlinear(ref: RefLib) -> dict:
    """assemble_nonlinear (nonlinear.cpp:11-107) on small meshes; coefficients U[-1, 1] from
    splitmix64 (problems.uniform01) with the seed stored next to each case."""
    out = {}
    meshes_ = [("square4", dgfem.unit_square_mesh(4, 0.15, 3, True, 4, 0).raw()),
               ("two_element", dict(mesh_cases())["two_element"])]
    for mname, raw in meshes_:
        mesh = ref.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
        n_el = raw["elements"].shape[0]
        for k in (1, 2, 3, 4):
            for qo in (0, 2 * k + 1):
                r = ref.reference(k, qo)
                nl = r.tables["n_local"]
                for rname, kind in REACTIONS.items():
                    seed = 1000 * k + 10 * qo + kind
                    coef = 2.0 * problems.uniform01(seed, n_el * nl) - 1.0
                    h, (ro, ci, va), _ = ref.assemble_nonlinear(mesh, r, coef, kind, threads=1)
                    name = f"{mname}_k{k}_q{qo}_{rname}"
                    out[f"{name}/coef"] = coef
                    out[f"{name}/seed"] = np.array(seed)
                    out[f"{name}/degree"] = np.array(k)
                    out[f"{name}/quad_order"] = np.array(qo)
                    out[f"{name}/kind"] = np.array(kind)
                    out[f"{name}/h"] = h
                    out[f"{name}/row_offsets"] = ro
                    out[f"{name}/cols"] = ci
                    out[f"{name}/vals"] = va
                    for kk, v in raw.items():
                        out[f"{name}/in_{kk}"] = np.asarray(v)
    # coefficient length check (test_nonlinear.cpp:55-65)
    raw = dict(meshes_)["square4"]
    mesh = ref.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
    try:
        ref.assemble_nonlinear(mesh, ref.reference(1, 0), np.zeros(7), capi.REACTION_SQUARE)
        status = 0
    except ReferenceError_ as e:
        status = e.status
    out["length_error/status"] = np.array(status)
    return out


def postprocess(ref: RefLib) -> dict:
    """l2_error / project / eval_solution (postprocess.cpp:14-93) of the reference on a jittered
    permuted 6x6 mesh, degrees 1..4, seeded coefficients and points."""
    out = {}
    m = dgfem.unit_square_mesh(6, 0.2, 8, True, 9)
    raw = m.raw()
    rmesh = ref.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
    for kk, v in raw.items():
        out[f"in_{kk}"] = np.asarray(v)
    exact = problems.function(capi.FN_SIN_SIN, (1.0,))
    f = problems.function(capi.FN_GAUSSIAN, (50.0, 0.5, 0.5))
    for k in (1, 2, 3, 4):
        rref = ref.reference(k, 0)
        nl = rref.tables["n_local"]
        coef = 2.0 * problems.uniform01(31 + k, m.n_elements * nl) - 1.0
        rng = np.random.default_rng(k)
        el = rng.integers(0, m.n_elements, 64).astype(np.int32)
        xh, yh = rng.random(64) * 0.5, rng.random(64) * 0.5
        out[f"k{k}/coef"] = coef
        out[f"k{k}/l2"] = np.array(ref.l2_error(rmesh, rref, coef, exact))
        out[f"k{k}/project"] = ref.project(rmesh, rref, f, m.n_elements)
        out[f"k{k}/el"], out[f"k{k}/xh"], out[f"k{k}/yh"] = el, xh, yh
        out[f"k{k}/eval"] = ref.eval_solution(coef, rref, el, xh, yh)
    return out


def refine(ref: RefLib) -> dict:
    """unit_square_mesh (mesh.cpp:189-211) and uniform_refine (mesh.cpp:153-187) of the
    reference: level 0 and level 4 arrays, all-Dirichlet and with Neumann sides 2|8."""
    out = {}
    for sides in (0, 2 | 8):
        for level in (0, 4):
            m = ref.unit_square_refined(level, sides)
            for k, v in m.arrays.items():
                out[f"s{sides}_l{level}/{k}"] = v
    return out


def main():
    ref = RefLib()
    which = sys.argv[1:] or ["tables", "meshes", "systems", "nonlinear", "postprocess", "refine"]
    makers = {"tables": tables, "meshes": meshes, "systems": systems, "nonlinear": nonlinear,
              "postprocess": postprocess, "refine": refine}
    for w in which:
        np.savez_compressed(os.path.join(HERE, f"{w}.npz"), **makers[w](ref))
        print(f"{w}.npz", os.path.getsize(os.path.join(HERE, f"{w}.npz")), "bytes")


if __name__ == "__main__":
    main()
