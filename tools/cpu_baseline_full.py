"""BASELINE.md §3's CPU-baseline protocol, run on the GPU box's host (tools only; the result
is committed as profiles/cpu_baseline_r02.json).

For each requested config: the reference's own `assemble_all` + `stiffness()` (oracle/_ref,
compiled from /root/reference/proj/src) on the config's FULL mesh and coefficients, with
Execution::parallel(nproc) and Execution::serial(); mesh construction (the reference's
build_mesh on the oracle/meshgen.py input) and ReferenceElement construction timed
separately; peak RSS of the child process.  Each (config, threads) runs in its own process so
the peak RSS is that run's.  No repo CUDA library is loaded.

    python tools/cpu_baseline_full.py 1 2 4 [--serial-max-elements N] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import os
import resource
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(cfg_index: int, threads: int, n: int | None) -> dict:
    from oracle import meshgen
    from oracle.oracle import RefLib
    from paper_1502_02941_b200 import problems
    cfg = problems.CONFIGS[cfg_index]
    lib = RefLib()
    t0 = time.perf_counter()
    raw = meshgen.config_raw(cfg, n)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    mesh = lib.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
    t_mesh = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = lib.reference(cfg.degree, cfg.quad_order)
    t_ref = time.perf_counter() - t0
    E = raw["elements"].shape[0]
    spec = problems.config_problem(cfg_index, E)
    clip = cfg.neumann_sides if cfg.neumann_inflow == 1 else 0
    runs = []
    for m in cfg.methods:
        p = lib.set_parameters(m, cfg.degree)
        p.sigma_interior, p.sigma_boundary = cfg.sigma, 2.0 * cfg.sigma
        p.neumann_inflow = cfg.neumann_inflow
        s = lib.assemble(mesh, ref, spec.c, p, threads=threads, clip_sides=clip)
        runs.append({"method": ["SIPG", "NIPG", "IIPG"][m], "assemble_all_s": s.seconds[0],
                     "stiffness_s": s.seconds[1]})
        del s
    total = sum(r["assemble_all_s"] + r["stiffness_s"] for r in runs)
    return {"config": cfg_index, "n": n or cfg.n, "elements": E, "threads": threads,
            "mesh_input_numpy_s": t_gen, "build_mesh_s": t_mesh, "reference_element_s": t_ref,
            "assemblies": runs, "elements_per_s": len(runs) * E / total,
            "peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", type=int, nargs="+")
    ap.add_argument("--serial-max-elements", type=int, default=600_000,
                    help="serial runs above this size use a halved mesh (time scales linearly)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cpu_baseline_full.json"))
    ap.add_argument("--child", nargs=3, type=int, help=argparse.SUPPRESS)
    a = ap.parse_args()
    if a.child:
        cfg_index, threads, n = a.child
        print(json.dumps(child(cfg_index, threads, n or None)), flush=True)
        return
    from paper_1502_02941_b200 import problems
    nproc = len(os.sched_getaffinity(0))
    cpu = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    out = {"cpu_model": cpu, "nproc": nproc, "runs": [],
           "protocol": "BASELINE.md §3: assemble_all + stiffness() of the reference (oracle/_ref), "
                       "P = nproc and P = 1, mesh / ReferenceElement construction separate, "
                       "peak RSS per process"}
    for c in a.configs:
        cfg = problems.CONFIGS[c]
        for threads in (nproc, 1):
            n = cfg.n
            if threads == 1:
                while 2 * n * n > a.serial_max_elements:
                    n //= 2
            cmd = [sys.executable, os.path.abspath(__file__), "0", "--child", str(c), str(threads),
                   str(n)]
            t0 = time.perf_counter()
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                out["runs"].append({"config": c, "threads": threads, "error": r.stderr[-500:]})
            else:
                rec = json.loads(r.stdout.strip().splitlines()[-1])
                rec["wall_s"] = time.perf_counter() - t0
                rec["full_config"] = n == cfg.n
                out["runs"].append(rec)
            print(json.dumps(out["runs"][-1]), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
