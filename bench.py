#!/usr/bin/env python
"""Benchmark of the B200 DG system assembly (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]
    python bench.py --op nonlinear [...]   # H(u), HJ(u) assembly

Workload (default): BASELINE.json configs[3] = config 4, the largest single-GPU config -- the
2048x2048 unit-square mesh (8,388,608 triangles, element numbering Fisher-Yates permuted), P1,
SIPG (sigma = 6), Gaussian manufactured solution.  One step = one assembly (K = D + C + R in BSR
form plus F, `assemble_all` + `stiffness()`).  `value` = elements assembled per second with
mesh, tables and coefficients resident in HBM; `e2e` = the same metric through the host-buffer
C-ABI call (dgb_assemble_all_host: H2D of the mesh, bind, assembly, D2H of K and F);
`secondary` = the other configs timed the same way in the same process (config 2 both as the
fused 3-method batch and as one launch per method).

Under torchrun (N > 1) each rank assembles its own shard (weak scaling; no collective on the
data path), the step time is the max over ranks.  `--impl reference` times the reference's
own CPU assembly (oracle/_ref, OpenMP on all host cores) on a bounded sample of the workload.
Other ops: --op nonlinear | solve | mesh | spmv | c1-throughput (see --help).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")
METRIC = "DG system assembly elements/sec (fp64, 1 B200) and achieved HBM GB/s vs roofline"
METRIC_NL = ("nonlinear reaction assembly H(u), HJ(u) elements/sec (fp64, 1 B200) and achieved "
             "HBM GB/s vs roofline")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=None,
                    help="BASELINE.json config (default 4: the largest single-GPU config, "
                         "8.4M triangles; --op solve defaults to config 1)")
    ap.add_argument("--secondary", default="2,2s,3,5,1",
                    help="assembly op, N = 1: also time these configs on the same box "
                         "(device-resident; 'Cs' = one launch per method instead of the fused "
                         "batch); '' for none")
    ap.add_argument("--op", choices=["assembly", "nonlinear", "solve", "mesh", "spmv",
                                     "c1-throughput"],
                    default="assembly",
                    help="assembly: the headline (assemble_all + stiffness); nonlinear: "
                         "assemble_nonlinear on the config's mesh and degree, r(u) = u^2; "
                         "solve: K x = F of the config's SIPG system (preconditioned GMRES); "
                         "mesh: build_mesh + uniform_refine to level --levels on the device; "
                         "spmv: config 4's 100 BSR SpMVs; c1-throughput: config 1 single "
                         "launch, CUDA-graph replay and --copies systems per launch")
    ap.add_argument("--precond", choices=["sgs", "jacobi"], default="sgs",
                    help="--op solve: GMRES preconditioner (multicolour block SGS or block Jacobi)")
    ap.add_argument("--copies", type=int, default=512, help="--op c1-throughput: systems per launch")
    ap.add_argument("--levels", type=int, default=10, help="--op mesh: refinement levels")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--minblocks", type=int, default=0, help="tuning knob (P2 kernel CTAs/SM)")
    ap.add_argument("--ablate", type=int, default=0,
                    help="profiling only, results wrong: skip kernel parts (see dg_assembly.cu)")
    ap.add_argument("--l2-policy", type=int, default=-1,
                    help="plan L2 policy bits (1: persist nodes, 2: evict-first output, 4: P1 load hints); "
                         "-1: the default for the config")
    ap.add_argument("--no-batch", action="store_true",
                    help="one dgb_assemble launch per method instead of one dgb_assemble_batch")
    ap.add_argument("--no-fuse", action="store_true",
                    help="batched launch with one CTA row per set (grid.y = methods) instead of "
                         "one per-element pass writing every set")
    ap.add_argument("--ws", type=int, default=-1,
                    help="warp-specialised kernel: 0 off, 1 default, 4..12 producer warps of 16")
    ap.add_argument("--p1-pipe", type=int, default=-1,
                    help="P1 pipelined persistent kernel: 0 off (one-shot kernel), 1 on (default)")
    ap.add_argument("--l2-carve-mb", type=int, default=0,
                    help="cap on the persisting-L2 carve-out of L2 policy bits 0/2 (MiB; tuning)")
    ap.add_argument("--no-bind", action="store_true",
                    help="recompute the BSR pattern in every assembly (count + scan launches)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def peak_hbm():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def algorithmic_bytes(mesh, nl: int, per_element_fields: int, sets: int = 1, world: int = 1) -> int:
    """every input read once, every output written once -- for a batched
    launch of `sets` parameter sets, the inputs once and the outputs once per set; a shard
    (world > 1) does 1/world of it.
    reads : 16 n_nodes + 12 E (elements) + 12 E (element_edges) + 8 n_edges (edge_elements)
            + 1 n_edges (edge_kind) + 8 E per per-element coefficient field
    writes: 8 nl^2 (E + 2I) (values) + 4 (E + 2I) (block cols) + 4 (E + 1) (row ptr)
            + 8 nl E (RHS)"""
    E, I, ne, nn = mesh.n_elements, mesh.n_interior_edges, mesh.n_edges, mesh.n_nodes
    nb = E + 2 * I
    reads = 16 * nn + 12 * E + 12 * E + 8 * ne + ne + 8 * E * per_element_fields
    writes = 8 * nl * nl * nb + 4 * nb + 4 * (E + 1) + 8 * nl * E
    return (reads + sets * writes) // world


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x1: "gpu_idle"}

    def __init__(self, device_index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _sample(self):
        p = self.nvml
        self.samples.append(p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM))
        try:
            mask = p.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            mask = p.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        for bit, name in self.REASONS.items():
            if mask & bit and name != "gpu_idle":
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            self._stop.wait(0.01)

    def __enter__(self):
        if self.nvml:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.nvml:
            self._stop.set()
            self.t.join()
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


_RAW_CACHE: dict = {}


def cpu_reference_sample(cfg_index: int, n_sample: int, seconds: float, threads: int = 0):
    """Times the reference's own assemble_all + stiffness() (oracle/_ref, OpenMP over `threads`
    host threads, default all) with config `cfg_index`'s coefficients on an n_sample^2
    unit-square mesh (the config's jitter / permutation / boundary tags), repeating until
    `seconds` of assembly time have accumulated (at least one assembly per method).  The mesh
    comes from oracle/meshgen.py (numpy) through the reference's own build_mesh, so this leg
    never loads the repo's CUDA library.  Falls back to the plain-C restatement when the
    reference library is absent.  Returns (elements/s, kind, cores, sample description,
    seconds)."""
    from oracle import meshgen
    from oracle import oracle as orc
    from paper_1502_02941_b200 import problems
    cfg = problems.CONFIGS[cfg_index]
    cores = threads if threads > 0 else _cores()
    key = (cfg_index, n_sample)
    if key not in _RAW_CACHE:
        _RAW_CACHE.clear()
        _RAW_CACHE[key] = {"raw": meshgen.config_raw(cfg, n_sample)}
    cache = _RAW_CACHE[key]
    raw = cache["raw"]
    E = raw["elements"].shape[0]
    spec = problems.config_problem(cfg_index, E)
    elements = 0
    t_total = 0.0
    try:
        lib = orc.RefLib()
        if "rmesh" not in cache:   # the reference's build_mesh (untimed, reported separately)
            t0 = time.perf_counter()
            cache["rmesh"] = lib.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"],
                                            raw["neumann"])
            cache["build_s"] = time.perf_counter() - t0
        params = []
        for m in cfg.methods:
            p = lib.set_parameters(m, cfg.degree)          # the reference's set_parameters
            p.sigma_interior, p.sigma_boundary = cfg.sigma, 2.0 * cfg.sigma
            p.neumann_inflow = cfg.neumann_inflow
            params.append(p)
        rmesh = cache["rmesh"]
        rref = lib.reference(cfg.degree, cfg.quad_order)
        kind = "reference"
        clip = cfg.neumann_sides if cfg.neumann_inflow == 1 else 0
        while True:
            for p in params:
                s = lib.assemble(rmesh, rref, spec.c, p, threads=cores, clip_sides=clip)
                t_total += s.seconds[0] + s.seconds[1]
                elements += E
                del s
            if t_total >= seconds:
                break
    except FileNotFoundError:
        from paper_1502_02941_b200 import dgfem   # fallback only: the port needs mesh arrays
        mesh = dgfem.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
        params = [dgfem.config_parameters(cfg, m) for m in cfg.methods]
        ol = orc.OracleLib()
        kind = "port"
        arrays, tables = mesh.arrays(), dgfem.ReferenceElement(cfg.degree, cfg.quad_order).tables()
        while True:
            for p in params:
                t0 = time.perf_counter()
                ol.assemble(arrays, tables, spec.c, p, threads=cores)
                t_total += time.perf_counter() - t0
                elements += E
            if t_total >= seconds:
                break
    full = " = the full config" if n_sample == cfg.n else ""
    desc = (f"config {cfg_index} on a {n_sample}x{n_sample} mesh ({E} elements{full}), "
            f"{len(cfg.methods)} method(s), assemble_all + stiffness() on {cores} threads, "
            f"{elements // E} assemblies in {t_total:.2f} s")
    return elements / t_total, kind, cores, desc, t_total


def cpu_sample_size(cfg_index: int, budget_s: float, threads: int = 0) -> int:
    """The largest n (the config's own n, halved until it fits) whose one-assembly-per-method
    reference time is estimated to fit `budget_s`, from a calibration on a 64 x 64 mesh (the
    reference's assembly time is linear in the element count)."""
    from paper_1502_02941_b200 import problems
    cfg = problems.CONFIGS[cfg_index]
    rate = cpu_reference_sample(cfg_index, 64, 0.3, threads)[0]   # elements/s
    n = cfg.n
    while n > 16 and len(cfg.methods) * 2 * n * n / rate > budget_s:
        n //= 2
    return n


def config_block(cfg, index: int, world: int, n_local: int) -> dict:
    """The bench line's `config`: identical for both arms (needs no CUDA library)."""
    E = 2 * cfg.n * cfg.n
    return {
        "workload": f"config {index}: {cfg.n}x{cfg.n} unit square, {E} triangles, P{cfg.degree}, "
                    "methods " + "/".join(["SIPG", "NIPG", "IIPG"][m] for m in cfg.methods)
                    + f", sigma={cfg.sigma:g}, quad_order {cfg.quad_order}",
        "elements_per_step": world * E * len(cfg.methods), "n_local": n_local,
        "global_mesh": f"{world * cfg.n}x{cfg.n} cells on [0,{world}]x[0,1]" if world > 1 else None,
        "l2": "flushed between timed steps by a 256 MiB write (outside the timed events)",
        "parallelism": f"{world} rank(s), element-row shards" if world > 1 else "1 GPU",
    }


def time_steps(run, stream, steps: int, warmup: int, flush, dist=None, clocks=None):
    """W untimed steps, then `steps` timed steps of a workload.ConfigRun: CUDA events on
    `stream` around every step and around every block-row kernel launch (recorded by the plan
    on the launching stream), L2 flushed between steps outside the events.  `clocks` (a
    ClockSampler) brackets the timed steps.  Returns (step_ms list, kernel_ms list)."""
    import torch
    for _ in range(warmup):
        flush.fill_(1.0)
        run.step(stream)
    run.check_status(stream)
    torch.cuda.synchronize()
    nk = run.launches_per_step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    kev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(nk)] for _ in range(steps)]
    for row in kev:  # torch creates the cudaEvent_t lazily: record once so .cuda_event exists
        for a, b in row:
            a.record(stream)
            b.record(stream)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    if clocks is not None:
        clocks.__enter__()
    for k in range(steps):
        flush.fill_(float(k))          # L2 flush between timed steps (outside the events)
        ev[k][0].record(stream)
        run.step(stream, kev[k])
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    if clocks is not None:
        clocks.__exit__(None, None, None)
    if dist:
        dist.barrier()
    run.check_status(stream)
    return ([a.elapsed_time(b) for a, b in ev],
            [a.elapsed_time(b) for row in kev for a, b in row])


def device_summary(run, step_ms, kern_ms, world: int = 1) -> dict:
    """Throughput and roofline figures of one timed ConfigRun (this rank's rows)."""
    sets = len(run.params) if run.batched else 1
    nbytes = algorithmic_bytes(run.mesh, run.ref.n_local, len(run.spec.per_element), sets, world)
    kms = sum(kern_ms) / len(kern_ms)
    ms = sum(step_ms) / len(step_ms)
    peak, _ = peak_hbm()
    achieved = nbytes / (kms / 1e3) / 1e9
    return {"value": round(len(run.params) * run.n_rows / (ms / 1e3), 1),
            "ms_per_step": round(ms, 4), "kernel_ms": round(kms, 4), "bytes_per_launch": nbytes,
            "achieved_gbs": round(achieved, 1), "frac": round(achieved / peak, 4),
            "kernel_share_of_step": round(sum(kern_ms) / sum(step_ms), 3)}


# ----------------------------------------------------------------------------- ours
def run_ours(args, world, rank, local):
    import torch
    from paper_1502_02941_b200 import capi, problems, workload

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = capi.load()
    cfg = problems.CONFIGS[args.config]
    options = {capi.OPTION_L2_POLICY: args.l2_policy,
               capi.OPTION_L2_CARVEOUT_MB: args.l2_carve_mb or None,
               capi.OPTION_MIN_BLOCKS: args.minblocks or None,
               capi.OPTION_PROFILE_ABLATE: args.ablate or None,
               capi.OPTION_BATCH_FUSE: 0 if args.no_fuse else None,
               capi.OPTION_WARP_SPECIALIZED: args.ws if args.ws >= 0 else None,
               capi.OPTION_P1_PIPELINE: args.p1_pipe if args.p1_pipe >= 0 else None}
    run = workload.ConfigRun(args.config, local, rank, world, batch=not args.no_batch,
                             bind=not args.no_bind, options=options)
    mesh, ref, spec = run.mesh, run.ref, run.spec
    batched = run.batched
    stream = torch.cuda.current_stream(local)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MiB > L2

    K = args.steps
    clocks = ClockSampler(local)
    step_ms, kern_ms = time_steps(run, stream, K, args.warmup, flush, dist, clocks)
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / K
    units_per_step = len(run.params) * mesh.n_elements   # all ranks together
    value = units_per_step * K / (total_ms / 1e3)
    launches = K * run.launches_per_step() * lib.dgb_plan_launch_count(run.plan._h)
    bind_ms = run.bind_ms

    # roofline of the block-row kernel (the dominant, and per step the only, launch)
    summ = device_summary(run, step_ms, kern_ms, world)
    peak, peak_kind = peak_hbm()
    traffic = None
    try:
        with open(PROFILE_SUMMARY) as f:
            entry = json.load(f).get(f"config{args.config}")
        if entry:
            traffic = entry.get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": summ["achieved_gbs"], "peak": peak, "unit": "GB/s",
                "frac": summ["frac"], "traffic": traffic, "peak_source": peak_kind,
                "kernel": kernel_name(ref.n_local, spec.c.advection.kind == capi.VEC_CONSTANT,
                                      batched, args),
                "kernel_ms": summ["kernel_ms"], "bytes_per_launch": summ["bytes_per_launch"],
                "assemblies_per_launch": len(run.params) if batched else 1,
                "kernel_share_of_step": summ["kernel_share_of_step"] if world == 1 else None}

    # e2e through the host-buffer C-ABI entry point (pinned host memory in and out)
    e2e = None
    if not args.no_e2e:
        from paper_1502_02941_b200 import dgfem
        local_mesh = mesh if world == 1 else dgfem.config_mesh(cfg)
        local_spec = spec if world == 1 else problems.config_problem(args.config, local_mesh.n_elements)
        e2e = run_e2e(args, local_mesh, ref, local_spec, run.params, local)
        if dist:
            t = torch.tensor([e2e["seconds"]], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["value"] = world * e2e["elements"] / float(t.item())
        e2e = {"value": round(e2e["value"], 1), "unit": "elements/s",
               "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
               "steps": e2e["steps"], "api": "dgb_assemble_all_host",
               "per_call": "H2D of mesh + coefficients, bind, assembly, D2H of K and F"}
    del run, mesh
    torch.cuda.empty_cache()

    # the other BASELINE configs on the same box, device-resident (N = 1 only)
    secondary = None
    if world == 1 and args.secondary:
        secondary = []
        for item in args.secondary.split(","):
            idx, batch = int(item.rstrip("s")), not item.endswith("s")   # "2s": one launch per method
            r2 = workload.ConfigRun(idx, local, batch=batch)
            s_ms, k_ms = time_steps(r2, stream, max(5, K // 2), 3, flush)
            d = {"config": idx, **device_summary(r2, s_ms, k_ms),
                 "launch": (f"one fused dgb_assemble_batch of {len(r2.params)} methods"
                            if r2.batched else f"one launch per method ({len(r2.params)})"),
                 "kernel": kernel_name(r2.ref.n_local,
                                       r2.spec.c.advection.kind == capi.VEC_CONSTANT,
                                       r2.batched, args),
                 "bind_ms": round(r2.bind_ms, 4)}
            secondary.append(d)
            del r2
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_sample = {1: 32, 2: 128, 3: 64, 4: 256, 5: 32}[args.config]
        v, kind, cores, desc, _ = cpu_reference_sample(args.config, n_sample, args.cpu_seconds)
        cpu = {"value": round(v, 1), "unit": "elements/s", "cores": cores, "kind": kind,
               "sample": desc}

    if dist:
        dist.destroy_process_group()
    if rank != 0:
        return
    conf = config_block(cfg, args.config, world, ref.n_local)
    conf.update({
        "nq_vol": ref.nq_vol, "nq_edge": ref.nq_edge,
        "l2_policy": l2_policy_text(args.l2_policy),
        "pattern": ("recomputed in every assembly (count + scan)" if args.no_bind else
                    "bound once per mesh (dgb_plan_bind_mesh: count + scan + adjacency; "
                    "untimed setup, see bind_ms); every assembly still writes row_ptr, block "
                    "columns, values and RHS"),
        "launch": ("one fused dgb_assemble_batch of the methods per step" if batched else
                   "one launch per method"),
    })
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "elements/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE.json config inputs; no dataset involved)",
        "config": conf,
        "bind_ms": round(bind_ms, 4) if bind_ms is not None else None,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "secondary": secondary,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def run_e2e(args, mesh, ref, spec, params, device):
    """dgb_assemble_all_host per method: H2D of the mesh + coefficient arrays from pinned host
    memory, plan setup, assembly, D2H of K (BSR) and F into pinned host memory."""
    import ctypes as C

    import torch
    from paper_1502_02941_b200 import capi, dgfem
    from paper_1502_02941_b200.capi import Bsr, MeshArrays

    lib = capi.load()
    pinned = {}
    for k, a in mesh.arrays().items():
        t = torch.from_numpy(a.copy()).pin_memory()
        pinned[k] = t
    mv = MeshArrays()
    mv.n_nodes, mv.n_elements, mv.n_edges = mesh.n_nodes, mesh.n_elements, mesh.n_edges
    mv.n_interior_edges = mesh.n_interior_edges
    for k, t in pinned.items():
        setattr(mv, k, t.data_ptr())
    prob = type(spec.c).from_buffer_copy(spec.c)
    keep = []
    for name, arr in spec.per_element.items():
        t = torch.from_numpy(arr).pin_memory()
        keep.append(t)
        getattr(prob, name).per_element = t.data_ptr()
    E, nl = mesh.n_elements, ref.n_local
    nnzb = lib.dgb_bsr_nnzb(E, mesh.n_interior_edges)
    rp = torch.empty(E + 1, dtype=torch.int32).pin_memory()
    col = torch.empty(nnzb, dtype=torch.int32).pin_memory()
    val = torch.empty(nnzb * nl * nl, dtype=torch.float64).pin_memory()
    rhs = torch.empty(E * nl, dtype=torch.float64).pin_memory()
    b = Bsr()
    b.n_block_rows, b.block_dim, b.nnzb = E, nl, nnzb
    b.row_ptr, b.col, b.val = rp.data_ptr(), col.data_ptr(), val.data_ptr()
    # (dgb_assemble_all_host uploads every mesh array except `edges`, which no device code reads)
    h2d = sum(t.numel() * t.element_size() for k, t in pinned.items() if k != "edges") + sum(
        t.numel() * t.element_size() for t in keep)
    d2h = rp.numel() * 4 + col.numel() * 4 + val.numel() * 8 + rhs.numel() * 8

    def one_step():
        for p in params:
            dgfem._check(lib.dgb_assemble_all_host(C.byref(mv), C.byref(ref.view), C.byref(prob),
                                                   C.byref(p), device, C.byref(b), rhs.data_ptr()))

    one_step()  # warm-up (module load, allocator)
    steps = max(2, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    secs = time.perf_counter() - t0
    elements = steps * len(params) * E
    return {"value": elements / secs, "seconds": secs, "elements": elements, "steps": steps,
            "h2d": h2d * len(params), "d2h": d2h * len(params)}



# ----------------------------------------------------------------------------- reference arm
def run_reference(args, world, rank):
    """The reference's own CPU assembly (oracle/_ref: assemble_all + stiffness(), OpenMP on
    every host core) on the same config, metric and unit as our arm.  Each step is one bounded
    sample: the config's own mesh when one assembly per method fits the per-step budget,
    otherwise the largest halving of it that does (the metric is per element, and the
    reference's time is linear in the element count).  Rank 0 only; the repo's CUDA library is
    never loaded (oracle/meshgen.py feeds the reference's build_mesh)."""
    if rank != 0:
        return
    from paper_1502_02941_b200 import problems
    cfg = problems.CONFIGS[args.config]
    per_step = max(0.5, min(10.0, 150.0 / max(1, args.steps + args.warmup)))
    n_sample = cpu_sample_size(args.config, per_step)
    for _ in range(args.warmup):
        cpu_reference_sample(args.config, n_sample, 0.0)
    vals, secs_total = [], 0.0
    kind = cores = desc = None
    for _ in range(args.steps):   # small samples repeat to ~1/4 of the step budget
        v, kind, cores, desc, secs = cpu_reference_sample(args.config, n_sample, 0.25 * per_step)
        vals.append(v)
        secs_total += secs
    value = len(vals) / sum(1.0 / v for v in vals)     # elements over total time
    conf = config_block(cfg, args.config, world, (cfg.degree + 1) * (cfg.degree + 2) // 2)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "elements/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * secs_total / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE.json config inputs; no dataset involved)",
        "config": conf,
        "sample": desc,
        "cpu_baseline": {"value": round(value, 1), "unit": "elements/s", "cores": cores,
                         "kind": kind, "sample": f"per step: {desc}"},
        "e2e": {"value": round(value, 1), "unit": "elements/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- nonlinear op
def nonlinear_bytes(mesh, nl: int) -> int:
    """Every input read once, every output written once: reads 16 n_nodes + 12 E (elements)
    + 8 nl E (coefficients); writes 8 nl E (H) + 8 nl^2 E (HJ blocks) + 4 E (block columns)
    + 4 (E + 1) (row pointer)."""
    E, nn = mesh.n_elements, mesh.n_nodes
    return 16 * nn + 12 * E + 8 * nl * E + 8 * nl * E + 8 * nl * nl * E + 4 * E + 4 * (E + 1)


def nonlinear_cpu_sample(cfg_index: int, n_sample: int, seconds: float):
    """The reference's assemble_nonlinear (oracle/_ref, OpenMP on all cores), else the C
    restatement, repeated on a bounded sample mesh for about `seconds`."""
    from oracle import oracle as orc
    from paper_1502_02941_b200 import capi, dgfem, problems
    cfg = problems.CONFIGS[cfg_index]
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    mesh = dgfem.unit_square_mesh(n_sample, cfg.jitter, problems.SEED_JITTER, cfg.permute,
                                  problems.SEED_PERMUTE, cfg.neumann_sides)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    coef = 2.0 * problems.uniform01(SEED_NL_COEF, mesh.n_elements * ref.n_local) - 1.0
    elements, t_total = 0, 0.0
    try:
        lib = orc.RefLib()
        raw = mesh.raw()
        rmesh = lib.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
        rref = lib.reference(cfg.degree, cfg.quad_order)
        kind = "reference"
        while True:
            _, _, secs = lib.assemble_nonlinear(rmesh, rref, coef, capi.REACTION_SQUARE, threads=cores)
            t_total += secs
            elements += mesh.n_elements
            if t_total >= seconds:
                break
    except FileNotFoundError:
        ol = orc.OracleLib()
        kind = "port"
        arrays, tables = mesh.arrays(), ref.tables()
        while True:
            t0 = time.perf_counter()
            ol.assemble_nonlinear(arrays, tables, coef, capi.REACTION_SQUARE, threads=cores)
            t_total += time.perf_counter() - t0
            elements += mesh.n_elements
            if t_total >= seconds:
                break
    desc = (f"P{cfg.degree} on a {n_sample}x{n_sample} unit-square mesh ({mesh.n_elements} "
            f"elements), r(u) = u^2, assemble_nonlinear x{elements // mesh.n_elements} in "
            f"{t_total:.1f} s")
    return elements / t_total, kind, cores, desc, t_total


SEED_NL_COEF = 0x5EED00F1


def run_nonlinear(args, world, rank, local):
    """assemble_nonlinear (nonlinear.cpp:11-107) on config `--config`'s mesh and degree with
    the registry's r(u) = u^2 (paper-boundary-layer) and seeded U[-1, 1] coefficients.  Each
    rank runs its own config-sized mesh (the op is element-local: weak scaling, no
    collective)."""
    import ctypes as C

    import torch
    from paper_1502_02941_b200 import capi, dgfem, problems

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = capi.load()
    cfg = problems.CONFIGS[args.config]
    mesh = dgfem.config_mesh(cfg)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    nl, E = ref.n_local, mesh.n_elements
    coef_np = 2.0 * problems.uniform01(SEED_NL_COEF, E * nl) - 1.0
    plan = dgfem.Plan(ref.view, local)
    dm = dgfem.DeviceMesh(mesh, local)
    coef = torch.from_numpy(coef_np).cuda(local)
    stream = torch.cuda.current_stream(local)
    if cfg.degree == 1:
        # P1: the plan bound to the mesh (as for the assembly): the kernel reads the vertices from
        # the bound geometry record instead of gathering nodes
        plan.bind_mesh(dm)
    h, hj = plan.assemble_nonlinear(dm, coef, capi.REACTION_SQUARE, stream=stream)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")

    def step():
        plan.assemble_nonlinear(dm, coef, capi.REACTION_SQUARE, h, hj, stream=stream)

    for _ in range(args.warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for k in range(K):
            flush.fill_(float(k))
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / K
    value = world * E * K / (total_ms / 1e3)
    nbytes = nonlinear_bytes(mesh, nl)
    achieved = nbytes / (ms / 1e3) / 1e9
    peak, peak_kind = peak_hbm()
    traffic = None
    try:
        with open(PROFILE_SUMMARY) as f:
            traffic = json.load(f).get(f"nonlinear_config{args.config}", {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_kind,
                "kernel": f"nonlinear_kernel<{nl}>", "kernel_ms": round(ms, 4),
                "bytes_per_launch": nbytes, "kernel_share_of_step": 1.0}

    e2e = None
    if not args.no_e2e:
        pin = {k: torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for k, a in mesh.arrays().items()}
        mv = capi.MeshArrays()
        mv.n_nodes, mv.n_elements, mv.n_edges = mesh.n_nodes, E, mesh.n_edges
        mv.n_interior_edges = mesh.n_interior_edges
        for k2, t2 in pin.items():
            setattr(mv, k2, t2.data_ptr())
        pc = torch.from_numpy(coef_np).pin_memory()
        ph = torch.empty(E * nl, dtype=torch.float64).pin_memory()
        prp = torch.empty(E + 1, dtype=torch.int32).pin_memory()
        pcol = torch.empty(E, dtype=torch.int32).pin_memory()
        pval = torch.empty(E * nl * nl, dtype=torch.float64).pin_memory()
        b = capi.Bsr()
        b.n_block_rows, b.block_dim, b.nnzb = E, nl, E
        b.row_ptr, b.col, b.val = prp.data_ptr(), pcol.data_ptr(), pval.data_ptr()
        r = capi.Reaction()
        r.kind = capi.REACTION_SQUARE

        def host_call():
            dgfem._check(lib.dgb_assemble_nonlinear_host(C.byref(mv), C.byref(ref.view), pc.data_ptr(),
                                                         E * nl, C.byref(r), local, ph.data_ptr(), C.byref(b)))
        host_call()
        steps = max(2, min(K, 10))
        t0 = time.perf_counter()
        for _ in range(steps):
            host_call()
        secs = time.perf_counter() - t0
        if dist:
            t = torch.tensor([secs], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            secs = float(t.item())
        h2d = 16 * mesh.n_nodes + 12 * E + 4 * 2 * mesh.n_edges + mesh.n_edges + 8 * E * nl
        e2e = {"value": round(world * E * steps / secs, 1), "unit": "elements/s",
               "h2d_bytes_per_step": 16 * mesh.n_nodes + 12 * E + 8 * E * nl,
               "d2h_bytes_per_step": 8 * E * nl + 4 * (E + 1) + 4 * E + 8 * E * nl * nl,
               "steps": steps, "api": "dgb_assemble_nonlinear_host"}
        del h2d
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, kind, cores, desc, _ = nonlinear_cpu_sample(args.config, 256, args.cpu_seconds)
        cpu = {"value": round(v, 1), "unit": "elements/s", "cores": cores, "kind": kind, "sample": desc}
    if dist:
        dist.destroy_process_group()
    if rank != 0:
        return
    line = {
        "metric": METRIC_NL, "value": round(value, 1), "unit": "elements/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded U[-1,1] coefficients on the config mesh; no dataset involved)",
        "config": {"workload": f"assemble_nonlinear, r(u) = u^2, config {args.config} mesh "
                               f"({cfg.n}x{cfg.n}, {E} triangles), P{cfg.degree}, nq_vol {ref.nq_vol}",
                   "elements_per_step": world * E, "n_local": nl,
                   "l2": "flushed between timed steps by a 256 MiB write (outside the timed events)",
                   "parallelism": f"{world} rank(s), one config mesh each" if world > 1 else "1 GPU"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": K * lib.dgb_plan_launch_count(plan._h),
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def run_reference_nonlinear(args, world, rank):
    if rank != 0:
        return
    per_step = max(0.5, min(10.0, 120.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        nonlinear_cpu_sample(args.config, 256, 0.0)
    vals, secs_total, kind, cores, desc = [], 0.0, None, None, None
    for _ in range(args.steps):
        v, kind, cores, desc, secs = nonlinear_cpu_sample(args.config, 256, per_step)
        vals.append(v)
        secs_total += secs
    value = statistics.fmean(vals)
    print(json.dumps({
        "impl": "reference", "metric": METRIC_NL, "value": round(value, 1), "unit": "elements/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * secs_total / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded U[-1,1] coefficients)",
        "config": {"workload": f"assemble_nonlinear (bounded CPU sample: {desc})",
                   "parallelism": f"OpenMP, {cores} host threads"},
        "cpu_baseline": {"value": round(value, 1), "unit": "elements/s", "cores": cores,
                         "kind": kind, "sample": desc},
        "e2e": {"value": round(value, 1), "unit": "elements/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


# ----------------------------------------------------------------------------- solve op
METRIC_SOLVE = "linear solve of the assembled DG system K x = F: unknowns/sec (fp64, 1 B200)"


def solve_bytes(E: int, nl: int, nnzb: int, iterations: int, restart: int,
                sgs: bool = False) -> int:
    """Modeled bytes of a preconditioned GMRES(m) solve, every operand read / written once per
    use: per Arnoldi step with k previous basis vectors -- SpMV (values, indices, x, y), the
    preconditioner (block Jacobi: inverse blocks, in, out; block SGS: two sweeps, each reading
    the off-diagonal blocks, the inverse diagonal blocks and the colour arrays), CGS2 (two passes
    of k+1 dots and a (k+1)-term update) and the normalisation."""
    n = E * nl
    spmv = 8 * nl * nl * nnzb + 4 * nnzb + 4 * (E + 1) + 16 * n
    if sgs:
        sweep = 8 * nl * nl * (nnzb - E) + 4 * nnzb + 4 * (E + 1) + 8 * nl * nl * E + 8 * E + 24 * n
        prec = 2 * sweep
    else:
        prec = 8 * nl * nl * E + 16 * n
    total = 0
    for j in range(iterations):
        k = j % restart
        cgs = 2 * ((k + 2) * 8 * n + (k + 1) * 8 * n + 16 * n)
        total += spmv + prec + cgs + 3 * 8 * n
    return total


def solve_cpu_sample(cfg_index: int, n_sample: int, seconds: float):
    """The reference's direct solve restated (oracle/newton.py: SuperLU standing in for Eigen's
    SparseLU, single-threaded) on a bounded sample of the config's system."""
    from oracle import newton as onewton
    from oracle.oracle import OracleLib, bsr_to_csr
    from paper_1502_02941_b200 import capi, dgfem, problems
    cfg = problems.CONFIGS[cfg_index]
    mesh = dgfem.unit_square_mesh(n_sample, cfg.jitter, problems.SEED_JITTER, cfg.permute,
                                  problems.SEED_PERMUTE, cfg.neumann_sides)
    spec = problems.config_problem(cfg_index, mesh.n_elements)
    tables = dgfem.ReferenceElement(cfg.degree, cfg.quad_order).tables()
    rp, col, val, rhs = OracleLib().assemble(mesh.arrays(), tables, spec.c,
                                             dgfem.config_parameters(cfg, capi.SIPG))
    ro, ci, va = bsr_to_csr(rp, col, val)
    F = rhs.reshape(-1)
    unknowns, t_total = 0, 0.0
    while True:
        t0 = time.perf_counter()
        onewton.direct_solve(ro, ci, va, F)
        t_total += time.perf_counter() - t0
        unknowns += F.size
        if t_total >= seconds:
            break
    desc = (f"SuperLU (stand-in for Eigen SparseLU, absent here) on the config {cfg_index} SIPG "
            f"system of a {n_sample}x{n_sample} mesh ({F.size} unknowns), "
            f"{unknowns // F.size} solves in {t_total:.1f} s")
    return unknowns / t_total, "port", 1, desc, t_total


def run_solve(args, world, rank, local):
    import torch
    from paper_1502_02941_b200 import capi, dgfem, problems
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = capi.load()
    cfg = problems.CONFIGS[args.config]
    mesh = dgfem.config_mesh(cfg)
    spec = problems.config_problem(args.config, mesh.n_elements)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    plan = dgfem.Plan(ref.view, local)
    dm, dp = dgfem.DeviceMesh(mesh, local), dgfem.DeviceProblem(spec, local)
    out = plan.assemble(dm, dp, dgfem.config_parameters(cfg, capi.SIPG), plan.allocate(dm))
    b = out.rhs.reshape(-1)
    n = b.numel()
    opts = dgfem.solve_options(preconditioner=capi.PRECOND_BLOCK_SGS if args.precond == "sgs"
                               else capi.PRECOND_BLOCK_JACOBI)
    pname = "multicolour block-SGS" if args.precond == "sgs" else "block-Jacobi"
    for _ in range(args.warmup):
        dgfem.solve(out, b, options=opts, device=local)
    torch.cuda.synchronize()
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    stream = torch.cuda.current_stream(local)
    infos = []
    if dist:
        dist.barrier()
    with ClockSampler(local) as clocks:
        for k in range(K):
            ev[k][0].record(stream)
            _, info = dgfem.solve(out, b, options=opts, device=local)   # synchronises
            ev[k][1].record(stream)
            infos.append(info)
        torch.cuda.synchronize()
    total_ms = sum(a.elapsed_time(bb) for a, bb in ev)
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / K
    value = world * n * K / (total_ms / 1e3)
    its = infos[-1]["iterations"]
    nbytes = solve_bytes(mesh.n_elements, ref.n_local, out.col.shape[0], its, opts.restart,
                         args.precond == "sgs")
    peak, peak_kind = peak_hbm()
    achieved = nbytes / (ms / 1e3) / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, kind, cores, desc, _ = solve_cpu_sample(args.config, {1: 32, 2: 48, 3: 16, 4: 128, 5: 16}[args.config],
                                                   args.cpu_seconds)
        cpu = {"value": round(v, 1), "unit": "unknowns/s", "cores": cores, "kind": kind, "sample": desc}
    if dist:
        dist.destroy_process_group()
    if rank != 0:
        return
    print(json.dumps({
        "metric": METRIC_SOLVE, "value": round(value, 1), "unit": "unknowns/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (the config's seeded SIPG system; no dataset involved)",
        "config": {"workload": f"dgb_solve of config {args.config}'s SIPG system ({n} unknowns, "
                               f"P{cfg.degree}), {pname} GMRES({opts.restart}), accepted under "
                               "direct_solve's bound 1e-10 (||A||_F ||x|| + ||b||)",
                   "iterations": its, "restarts": infos[-1]["restarts"],
                   "defect_norm2": infos[-1]["defect_norm2"], "bound": infos[-1]["bound"],
                   "parallelism": "1 GPU" if world == 1 else f"{world} independent replicas"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_kind,
                     "kernel": f"whole solve (modeled bytes: SpMV + {pname} + CGS2 per step)",
                     "kernel_ms": round(ms, 3), "bytes_per_launch": nbytes},
        "cpu_baseline": cpu,
        "e2e": None,
        "gpu_launches": None,
        "clocks": clocks.summary(),
    }), flush=True)


# ----------------------------------------------------------------------------- spmv op
METRIC_SPMV = ("BSR SpMV y = K x of the assembled config-4 system (fp64, 1 B200): block rows/sec "
               "and achieved HBM GB/s vs roofline")


def spmv_cpu_sample(n_sample: int, seconds: float):
    """The reference's own matvec (sparse.cpp:116-129: serial CSR loop over stiffness()) on
    config 4's system over an n_sample^2 mesh (oracle/_ref via ref_shim, which adds a copy of x
    in and y out per call); the C restatement's OpenMP product when the reference is absent.
    Returns (block rows/s, kind, cores, description)."""
    from oracle import meshgen
    from oracle import oracle as orc
    from paper_1502_02941_b200 import capi, problems
    cfg = problems.CONFIGS[4]
    raw = meshgen.config_raw(cfg, n_sample)
    E = raw["elements"].shape[0]
    x = 2.0 * problems.uniform01(problems.SEED_SPMV_X, 3 * E) - 1.0
    y = np.zeros(3 * E)
    lib = orc.RefLib()
    p = lib.set_parameters(capi.SIPG, 1)
    p.sigma_interior, p.sigma_boundary = cfg.sigma, 2.0 * cfg.sigma
    rmesh = lib.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
    system = lib.assemble(rmesh, lib.reference(1, cfg.quad_order), problems.config_problem(4).c, p)
    reps, t = 0, 0.0
    while t < seconds:
        t0 = time.perf_counter()
        system.matvec(x, y)
        t += time.perf_counter() - t0
        reps += 1
    desc = (f"the reference's matvec on config 4's SIPG system over a {n_sample}x{n_sample} mesh "
            f"({E} block rows), {reps} products in {t:.2f} s, serial")
    return E * reps / t, "reference", 1, desc


def run_spmv(args, world, rank, local):
    """Config 4's 100 BSR SpMVs (BASELINE.json configs[3]) on the matrix the bench's assembly
    produces.  One step = the 100 products y = K x with x seeded U[-1, 1]; the matrix (2.4 GB)
    and x (201 MB) exceed L2, so no flush is needed between products.  `value` = block rows
    multiplied per second; roofline per product = SURVEY.md §8(d)'s 2,985,721,860 B."""
    import torch
    from paper_1502_02941_b200 import workload
    torch.cuda.set_device(local)
    sp = workload.SpmvRun(4, local)
    stream = torch.cuda.current_stream(local)
    n_prod = 100
    for _ in range(args.warmup):
        for _ in range(n_prod):
            sp.step(stream)
    torch.cuda.synchronize()
    K = args.steps
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(n_prod)] for _ in range(K)]
    clocks = ClockSampler(local)
    with clocks:
        for k in range(K):
            for j in range(n_prod):
                ev[k][j][0].record(stream)
                sp.step(stream)
                ev[k][j][1].record(stream)
        torch.cuda.synchronize()
    prod_ms = [a.elapsed_time(b) for row in ev for a, b in row]
    step_ms = [sum(a.elapsed_time(b) for a, b in row) for row in ev]
    E = sp.run.n_rows
    ms = sum(step_ms) / K
    value = n_prod * E / (ms / 1e3)
    nbytes = sp.bytes_per_product()
    avg = sum(prod_ms) / len(prod_ms)
    peak, peak_kind = peak_hbm()
    traffic = None
    try:
        with open(PROFILE_SUMMARY) as f:
            traffic = json.load(f).get("spmv_config4", {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    e2e = None
    if not args.no_e2e:   # host x in, host y out, per product, through the C-ABI product
        hx = sp.x.cpu().pin_memory()
        hy = torch.empty_like(hx).pin_memory()
        dx, dy = torch.empty_like(sp.x), torch.empty_like(sp.y)
        torch.cuda.synchronize()
        reps = 10
        t0 = time.perf_counter()
        for _ in range(reps):
            dx.copy_(hx, non_blocking=True)
            sp.x, x_keep = dx, sp.x
            sp.step(stream, dy)
            sp.x = x_keep
            hy.copy_(dy, non_blocking=True)
            torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        e2e = {"value": round(reps * E / secs, 1), "unit": "block rows/s",
               "h2d_bytes_per_step": hx.numel() * 8, "d2h_bytes_per_step": hy.numel() * 8,
               "note": "per product: H2D of x, dgb_spmv, D2H of y (K resident)"}
    cpu = None
    if not args.no_cpu_baseline:
        try:
            v, kind, cores, desc = spmv_cpu_sample(512, min(args.cpu_seconds, 10.0))
            cpu = {"value": round(v, 1), "unit": "block rows/s", "cores": cores, "kind": kind,
                   "sample": desc}
        except FileNotFoundError:
            cpu = None
    print(json.dumps({
        "metric": METRIC_SPMV, "value": round(value, 1), "unit": "block rows/s", "n_gpus": 1,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (config 4's assembled system, x seeded U[-1,1])",
        "config": {"workload": f"config 4: {n_prod} BSR SpMVs per step on the 2048x2048 P1 SIPG "
                               f"matrix ({E} block rows, {sp.system.col.shape[0]} 3x3 blocks)",
                   "l2": "matrix 2.4 GB and x 201 MB exceed L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "achieved": round(nbytes / (avg / 1e3) / 1e9, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(nbytes / (avg / 1e3) / 1e9 / peak, 4),
                     "traffic": traffic, "peak_source": peak_kind,
                     "kernel": "bsr_spmv_kernel<3,128,3>", "kernel_ms": round(avg, 4),
                     "bytes_per_launch": nbytes, "kernel_share_of_step": 1.0},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": K * n_prod,
        "clocks": clocks.summary(),
    }), flush=True)


# ----------------------------------------------------------------------------- small-config throughput
def run_c1_throughput(args, world, rank, local):
    """Config 1's throughput figures (BASELINE.md §2 note 1): config 1 (2,048 triangles, 0.77 MB
    of output) cannot approach its roofline in one launch, so beside the single launch this
    reports (a) a CUDA graph replaying G single assemblies back to back and (b) B = --copies
    independent config-1 systems in ONE launch of the bound block-row kernel (the disjoint
    union of B copies of the mesh; workload.BatchedSystemsRun).  `value` = (b)'s elements/s."""
    import torch
    from paper_1502_02941_b200 import workload
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream(local)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")
    K = args.steps
    single = workload.ConfigRun(1, local)
    s_ms, k_ms = time_steps(single, stream, K, args.warmup, flush)
    single_sum = device_summary(single, s_ms, k_ms)
    G = 100
    graph = workload.capture_graph(single, G)
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        flush.fill_(float(k))
        gev[k][0].record(stream)
        graph.replay()
        gev[k][1].record(stream)
    torch.cuda.synchronize()
    g_ms = sum(a.elapsed_time(b) for a, b in gev) / K
    E1 = single.n_rows
    del graph, single
    torch.cuda.empty_cache()
    batch = workload.BatchedSystemsRun(1, args.copies, local)
    clocks = ClockSampler(local)
    b_ms, bk_ms = time_steps(batch, stream, K, args.warmup, flush, clocks=clocks)
    summ = device_summary(batch, b_ms, bk_ms)
    bind_ms, launches_per_step, n_rows_batch = batch.bind_ms, batch.launches_per_step(), batch.n_rows
    peak, peak_kind = peak_hbm()
    # the same launch over 8x as many systems (launch ramp and tail amortised further)
    larger = None
    if args.copies * 8 * E1 <= 16 * 1024 * 1024:
        del batch
        torch.cuda.empty_cache()
        big = workload.BatchedSystemsRun(1, args.copies * 8, local)
        g_ms2, gk_ms2 = time_steps(big, stream, K, args.warmup, flush)
        s2 = device_summary(big, g_ms2, gk_ms2)
        larger = {"copies": args.copies * 8, "value": s2["value"], "kernel_ms": s2["kernel_ms"],
                  "ms_per_step": s2["ms_per_step"], "frac": s2["frac"]}
        batch = big
    print(json.dumps({
        "metric": METRIC + " -- config 1 throughput (many systems)", "value": summ["value"],
        "unit": "elements/s", "n_gpus": 1, "steps": K, "warmup": args.warmup,
        "ms_per_step": summ["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (config 1's seeded inputs, replicated)",
        "config": {"workload": f"{args.copies} independent config-1 systems (32x32 unit square, "
                               f"2048 triangles, P1, SIPG) per launch: the bound block-row kernel "
                               f"over their disjoint union ({n_rows_batch} block rows)",
                   "l2": "flushed between timed steps by a 256 MiB write (outside the timed events)"},
        "roofline": {"bound": "hbm", "achieved": summ["achieved_gbs"], "peak": peak, "unit": "GB/s",
                     "frac": summ["frac"], "traffic": None, "peak_source": peak_kind,
                     "kernel": "assemble_p1_pipe_kernel", "kernel_ms": summ["kernel_ms"],
                     "bytes_per_launch": summ["bytes_per_launch"],
                     "kernel_share_of_step": summ["kernel_share_of_step"]},
        "single_launch": {"value": single_sum["value"], "kernel_ms": single_sum["kernel_ms"],
                          "ms_per_step": single_sum["ms_per_step"], "frac": single_sum["frac"]},
        "graph_replay": {"assemblies_per_replay": G, "ms_per_replay": round(g_ms, 4),
                         "us_per_assembly": round(1e3 * g_ms / G, 2),
                         "value": round(G * E1 / (g_ms / 1e3), 1)},
        "larger_batch": larger,
        "bind_ms": round(bind_ms, 4),
        "cpu_baseline": None, "e2e": None,
        "gpu_launches": K * launches_per_step,
        "clocks": clocks.summary(),
    }), flush=True)


# ----------------------------------------------------------------------------- mesh op
METRIC_MESH = ("mesh topology build (build_mesh + uniform_refine chain to the C4 size): "
               "elements/sec (1 B200)")


def run_mesh(args, world, rank, local):
    """uniform_refine from the reference's unit_square_mesh (8 triangles) to --levels (10: 8.4M
    triangles, the reference's C4 mesh), every level through the device build_mesh.  `value` =
    elements of the final level / the time of the whole chain.  cpu_baseline = the reference's
    own uniform_refine chain (oracle/_ref) to a bounded level, rescaled to elements/s."""
    import torch
    from paper_1502_02941_b200 import capi, dgfem
    torch.cuda.set_device(local)
    base = {"nodes": np.array([[0.0, 0.0], [0.5, 0.0], [1.0, 0.0], [0.0, 0.5], [0.5, 0.5], [1.0, 0.5],
                               [0.0, 1.0], [0.5, 1.0], [1.0, 1.0]]),
            "elements": np.array([[3, 0, 4], [0, 1, 4], [4, 1, 5], [1, 2, 5], [6, 3, 7], [3, 4, 7],
                                  [7, 4, 8], [4, 5, 8]], np.int32),
            "dirichlet": np.array([[0, 1], [1, 2], [0, 3], [2, 5], [3, 6], [5, 8], [6, 7], [7, 8]], np.int32),
            "neumann": np.zeros((0, 2), np.int32)}   # unit_square_mesh() (mesh.cpp:189-211)

    def chain():
        m = dgfem.device_build_mesh(base["nodes"], base["elements"], base["dirichlet"], base["neumann"], local)
        for _ in range(args.levels):
            m = m.refine()
        return m
    for _ in range(args.warmup):
        chain()
    torch.cuda.synchronize()
    K = args.steps
    times = []
    with ClockSampler(local) as clocks:
        for _ in range(K):
            t0 = time.perf_counter()      # the chain synchronises at every level (host counts)
            m = chain()
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
    sec = sum(times) / K
    E = m.n_elements
    value = E / sec
    cpu = None
    if not args.no_cpu_baseline:
        try:
            from oracle import oracle as orc
            lib = orc.RefLib()
            lvl = min(args.levels, 8)
            t0 = time.perf_counter()
            lib.unit_square_refined(lvl, 0)
            t = time.perf_counter() - t0
            e_cpu = 8 * 4 ** lvl
            cpu = {"value": round(e_cpu / t, 1), "unit": "elements/s", "cores": 1, "kind": "reference",
                   "sample": f"the reference's unit_square_mesh + uniform_refine x{lvl} ({e_cpu} "
                             f"elements) in {t:.2f} s (includes the ref_shim flatten copy)"}
        except FileNotFoundError:
            cpu = None
    print(json.dumps({
        "metric": METRIC_MESH, "value": round(value, 1), "unit": "elements/s", "n_gpus": 1,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(1e3 * sec, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (the reference's unit_square_mesh, refined)",
        "config": {"workload": f"device build_mesh of unit_square_mesh() + {args.levels} x "
                               f"uniform_refine (each level rebuilt by the device build_mesh): "
                               f"{E} triangles, {m.n_edges} edges",
                   "timing": "host wall clock around the chain (it synchronises per level)"},
        "roofline": None, "cpu_baseline": cpu, "e2e": None, "gpu_launches": None,
        "clocks": clocks.summary(),
    }), flush=True)


def kernel_name(nl: int, const_b: bool, batched: bool, args) -> str:
    """The block-row kernel the library launches for this run (dg_assembly.cu launch_v2)."""
    bound = not args.no_bind
    if nl == 3 and const_b:
        return "assemble_p1_pipe_kernel" if bound and args.p1_pipe != 0 else "assemble_p1_kernel"
    if nl == 6 and const_b and bound and args.ws != 0 and ((batched and not args.no_fuse) or args.ws > 1):
        return "assemble_ws_kernel"
    return f"assemble_kernel<{nl}>"


def l2_policy_text(l2: int) -> str:
    """The bench line's description of DGB_OPTION_L2_POLICY (include/dgfem_b200.h)."""
    if l2 < 0:
        return "auto (library default per kernel)"
    parts = [t for bit, t in ((1, "node coordinates persisting in L2"), (2, "evict-first output"),
                              (4, "load hints: node gathers evict-last, records evict-first"))
             if l2 & bit]
    return " + ".join(parts) or "default"


def main():
    args = parse_args()
    if args.config is None:
        args.config = 1 if args.op == "solve" else 4
    world, rank, local = dist_setup(args)
    if args.op == "mesh":
        if rank == 0:
            run_mesh(args, world, rank, local)
        return
    if args.op == "solve":
        run_solve(args, world, rank, local)
        return
    if args.op == "spmv":
        if rank == 0:
            run_spmv(args, world, rank, local)
        return
    if args.op == "c1-throughput":
        if rank == 0:
            run_c1_throughput(args, world, rank, local)
        return
    if args.op == "nonlinear":
        if args.impl == "reference":
            run_reference_nonlinear(args, world, rank)
        else:
            run_nonlinear(args, world, rank, local)
    elif args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
