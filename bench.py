#!/usr/bin/env python
"""Benchmark of the B200 DG system assembly (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]
    python bench.py --op nonlinear [...]   # H(u), HJ(u) assembly

Workload (default): BASELINE.json configs[1] = config 2 -- the 256x256 unit-square mesh
(131,072 triangles), P2, assembled with each of SIPG, NIPG and IIPG (sigma = 18).  One step =
the three assemblies (K = D + C + R in BSR form plus F).  `value` = elements assembled per
second with mesh, tables and coefficients resident in HBM; `e2e` = the same metric through
the host-buffer C-ABI call (dgb_assemble_all_host: H2D of the mesh, assembly, D2H of K and F).

Under torchrun (N > 1) each rank assembles its own shard (weak scaling; no collective on the
data path), the step time is the max over ranks.  `--impl reference` times the reference's
own CPU assembly (oracle/_ref, OpenMP on all host cores) on a bounded sample of the workload.
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
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--op", choices=["assembly", "nonlinear", "solve", "mesh"], default="assembly",
                    help="assembly: the headline (assemble_all + stiffness); nonlinear: "
                         "assemble_nonlinear on the config's mesh and degree, r(u) = u^2; "
                         "solve: K x = F of the config's SIPG system (block-Jacobi GMRES); "
                         "mesh: build_mesh + uniform_refine to level --levels on the device")
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


def cpu_reference_sample(cfg_index: int, n_sample: int, seconds: float):
    """Times the reference's own assemble_all + stiffness() (oracle/_ref, OpenMP on every host
    core) on config `cfg_index`'s coefficients over an n_sample^2 unit-square mesh; falls back
    to the plain-C restatement when the reference library is absent.  Returns
    (elements/s, kind, cores, sample description, seconds)."""
    from oracle import oracle as orc
    from paper_1502_02941_b200 import dgfem, problems
    cfg = problems.CONFIGS[cfg_index]
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    mesh = dgfem.unit_square_mesh(n_sample, cfg.jitter, problems.SEED_JITTER, cfg.permute,
                                  problems.SEED_PERMUTE, cfg.neumann_sides)
    spec = problems.config_problem(cfg_index, mesh.n_elements)
    params = [dgfem.config_parameters(cfg, m) for m in cfg.methods]
    elements = 0
    t_total = 0.0
    try:
        lib = orc.RefLib()
        raw = mesh.raw()
        rmesh = lib.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
        rref = lib.reference(cfg.degree, cfg.quad_order)
        kind = "reference"
        clip = cfg.neumann_sides if cfg.neumann_inflow == 1 else 0
        while True:
            for p in params:
                s = lib.assemble(rmesh, rref, spec.c, p, threads=cores, clip_sides=clip)
                t_total += s.seconds[0] + s.seconds[1]
                elements += mesh.n_elements
                del s
            if t_total >= seconds:
                break
    except FileNotFoundError:
        ol = orc.OracleLib()
        kind = "port"
        arrays, tables = mesh.arrays(), dgfem.ReferenceElement(cfg.degree, cfg.quad_order).tables()
        while True:
            for p in params:
                t0 = time.perf_counter()
                ol.assemble(arrays, tables, spec.c, p, threads=cores)
                t_total += time.perf_counter() - t0
                elements += mesh.n_elements
            if t_total >= seconds:
                break
    desc = (f"config {cfg_index} coefficients on a {n_sample}x{n_sample} unit-square mesh "
            f"({mesh.n_elements} elements), methods {len(params)}, assemble_all + stiffness(), "
            f"{elements // mesh.n_elements} assemblies in {t_total:.1f} s")
    return elements / t_total, kind, cores, desc, t_total


# ----------------------------------------------------------------------------- ours
def run_ours(args, world, rank, local):
    import ctypes as C

    import torch
    from paper_1502_02941_b200 import capi, dgfem, problems

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = capi.load()
    from paper_1502_02941_b200 import shard
    cfg = problems.CONFIGS[args.config]
    mesh = dgfem.config_mesh(cfg, strips=world)       # global mesh: world x config size
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(args.config, mesh.n_elements)
    params = [dgfem.config_parameters(cfg, m) for m in cfg.methods]
    begin, end = shard.row_range(mesh.n_elements, rank, world)
    l2 = args.l2_policy  # -1: the library's per-kernel default (profiles/NOTES.md)
    shards = [shard.ShardAssembler(mesh, ref, spec, local, begin, end, bind=False)]
    shards[0].plan.set_option(capi.OPTION_L2_POLICY, l2)
    if args.l2_carve_mb:  # read at bind time
        shards[0].plan.set_option(capi.OPTION_L2_CARVEOUT_MB, args.l2_carve_mb)
    if not args.no_bind:
        shards[0].plan.bind_mesh(shards[0].dmesh, begin, end)
    shards += [shard.ShardAssembler(mesh, ref, spec, local, begin, end, share=shards[0])
               for _ in params[1:]]   # one plan and one device mesh for all methods
    plan = shards[0].plan
    if args.minblocks:
        plan.set_option(capi.OPTION_MIN_BLOCKS, args.minblocks)
    if args.ablate:
        plan.set_option(capi.OPTION_PROFILE_ABLATE, args.ablate)
    if args.no_fuse:
        plan.set_option(capi.OPTION_BATCH_FUSE, 0)
    if args.ws >= 0:
        plan.set_option(capi.OPTION_WARP_SPECIALIZED, args.ws)
    if args.p1_pipe >= 0:
        plan.set_option(capi.OPTION_P1_PIPELINE, args.p1_pipe)
    stream = torch.cuda.current_stream(local)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MiB > L2

    batched = (not args.no_batch) and len(params) > 1

    def step(kernel_events=None):
        if batched:  # one dgb_assemble_batch: all methods in one launch when the rows are bound
            if kernel_events is not None:
                ks, ke = kernel_events[0]
                lib.dgb_plan_set_kernel_events(plan._h, C.c_void_p(ks.cuda_event), C.c_void_p(ke.cuda_event))
            shard.assemble_batch(shards, params, stream=stream, check=False)
        else:
            for i, (p, sh) in enumerate(zip(params, shards)):
                if kernel_events is not None:
                    ks, ke = kernel_events[i]
                    lib.dgb_plan_set_kernel_events(plan._h, C.c_void_p(ks.cuda_event), C.c_void_p(ke.cuda_event))
                sh.assemble(p, stream=stream, check=False)
        lib.dgb_plan_set_kernel_events(plan._h, None, None)

    for _ in range(args.warmup):
        flush.fill_(1.0)
        step()
    dgfem._check(lib.dgb_plan_status(plan._h, C.c_void_p(stream.cuda_stream)))
    torch.cuda.synchronize()

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    kev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in params] for _ in range(K)]
    for row in kev:  # torch creates the cudaEvent_t lazily: record once so .cuda_event exists
        for a, b in row:
            a.record(stream)
            b.record(stream)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for k in range(K):
            flush.fill_(float(k))          # L2 flush between timed steps (outside the events)
            ev[k][0].record(stream)
            step(kev[k])
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    dgfem._check(lib.dgb_plan_status(plan._h, C.c_void_p(stream.cuda_stream)))
    step_ms = [a.elapsed_time(b) for a, b in ev]
    kern_ms = [a.elapsed_time(b) for row in kev for a, b in (row[:1] if batched else row)]
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / K
    units_per_step = len(params) * mesh.n_elements   # all ranks together
    value = units_per_step * K / (total_ms / 1e3)

    # roofline of the block-row kernel (dominant launch)
    per_elem_fields = len(spec.per_element)
    sets_per_launch = len(params) if batched else 1
    bytes_per_launch = algorithmic_bytes(mesh, ref.n_local, per_elem_fields, sets_per_launch, world)
    kern_avg_ms = sum(kern_ms) / len(kern_ms)
    achieved = bytes_per_launch / (kern_avg_ms / 1e3) / 1e9
    peak, peak_kind = peak_hbm()
    traffic = None
    try:
        with open(PROFILE_SUMMARY) as f:
            prof = json.load(f)
        entry = prof.get(f"config{args.config}")
        if entry:
            traffic = entry.get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "peak_source": peak_kind,
                "kernel": kernel_name(ref.n_local, spec.c.advection.kind == capi.VEC_CONSTANT, batched, args),
                "kernel_ms": round(kern_avg_ms, 4), "bytes_per_launch": bytes_per_launch,
                "assemblies_per_launch": sets_per_launch,
                "kernel_share_of_step": round(sum(kern_ms) / total_ms, 3) if world == 1 else None}

    # e2e through the host-buffer C-ABI entry point (pinned host memory in and out)
    e2e = None
    if not args.no_e2e:
        local_mesh = mesh if world == 1 else dgfem.config_mesh(cfg)
        local_spec = spec if world == 1 else problems.config_problem(args.config, local_mesh.n_elements)
        e2e = run_e2e(args, local_mesh, ref, local_spec, params, local)
        if dist:
            t = torch.tensor([e2e["seconds"]], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["value"] = world * e2e["elements"] / float(t.item())
        e2e = {"value": round(e2e["value"], 1), "unit": "elements/s",
               "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
               "steps": e2e["steps"], "api": "dgb_assemble_all_host"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_sample = {1: 32, 2: 96, 3: 32, 4: 128, 5: 24}[args.config]
        v, kind, cores, desc, secs = cpu_reference_sample(args.config, n_sample, args.cpu_seconds)
        cpu = {"value": round(v, 1), "unit": "elements/s", "cores": cores, "kind": kind,
               "sample": desc}

    if dist:
        dist.destroy_process_group()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "elements/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE.json config inputs; no dataset involved)",
        "config": {
            "workload": f"config {args.config}: {cfg.n}x{cfg.n} unit square, {mesh.n_elements} "
                        f"triangles, P{cfg.degree}, methods "
                        + "/".join(["SIPG", "NIPG", "IIPG"][m] for m in cfg.methods)
                        + f", sigma={cfg.sigma:g}",
            "elements_per_step": units_per_step, "n_local": ref.n_local,
            "global_mesh": f"{world * cfg.n}x{cfg.n} cells on [0,{world}]x[0,1]" if world > 1 else None,
            "nq_vol": ref.nq_vol, "nq_edge": ref.nq_edge,
            "l2": "flushed between timed steps by a 256 MiB write (outside the timed events)",
            "l2_policy": l2_policy_text(l2),
            "pattern": ("recomputed in every assembly (count + scan)" if args.no_bind else
                        "bound once per mesh (dgb_plan_bind_mesh, untimed setup); every assembly "
                        "still writes row_ptr, block columns, values and RHS"),
            "parallelism": f"{world} rank(s), element-row shards" if world > 1 else "1 GPU",
            "launch": ("one dgb_assemble_batch per step (the methods as grid.y of one launch when "
                       "the P2 tensor-core kernel applies)" if batched else "one launch per method"),
        },
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": K * (1 if batched else len(params)) * lib.dgb_plan_launch_count(plan._h),
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
    h2d = sum(t.numel() * t.element_size() for t in pinned.values()) + sum(
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
    if rank != 0:
        return
    from paper_1502_02941_b200 import problems
    cfg = problems.CONFIGS[args.config]
    n_sample = {1: 32, 2: 64, 3: 24, 4: 96, 5: 16}[args.config]
    per_step = max(0.5, min(10.0, 120.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_reference_sample(args.config, n_sample, 0.0)
    vals, secs_total = [], 0.0
    kind = cores = desc = None
    for _ in range(args.steps):
        v, kind, cores, desc, secs = cpu_reference_sample(args.config, n_sample, per_step)
        vals.append(v)
        secs_total += secs
    value = statistics.fmean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "elements/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * secs_total / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE.json config inputs)",
        "config": {"workload": f"config {args.config} (bounded CPU sample: {desc})",
                   "parallelism": f"OpenMP, {cores} host threads"},
        "cpu_baseline": {"value": round(value, 1), "unit": "elements/s", "cores": cores,
                         "kind": kind, "sample": desc},
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


def solve_bytes(E: int, nl: int, nnzb: int, iterations: int, restart: int) -> int:
    """Modeled bytes of a block-Jacobi GMRES(m) solve, every operand read / written once per
    use: per Arnoldi step with k previous basis vectors -- SpMV (values, indices, x, y),
    block-Jacobi apply (inverse blocks, in, out), CGS2 (two passes of k+1 dots and a
    (k+1)-term update) and the normalisation."""
    n = E * nl
    spmv = 8 * nl * nl * nnzb + 4 * nnzb + 4 * (E + 1) + 16 * n
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
    opts = dgfem.solve_options()
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
    nbytes = solve_bytes(mesh.n_elements, ref.n_local, out.col.shape[0], its, opts.restart)
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
                               f"P{cfg.degree}), block-Jacobi GMRES({opts.restart}), accepted under "
                               "direct_solve's bound 1e-10 (||A||_F ||x|| + ||b||)",
                   "iterations": its, "restarts": infos[-1]["restarts"],
                   "defect_norm2": infos[-1]["defect_norm2"], "bound": infos[-1]["bound"],
                   "parallelism": "1 GPU" if world == 1 else f"{world} independent replicas"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_kind,
                     "kernel": "whole solve (modeled bytes: SpMV + block-Jacobi + CGS2 per step)",
                     "kernel_ms": round(ms, 3), "bytes_per_launch": nbytes},
        "cpu_baseline": cpu,
        "e2e": None,
        "gpu_launches": None,
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
    world, rank, local = dist_setup(args)
    if args.op == "mesh":
        if rank == 0:
            run_mesh(args, world, rank, local)
        return
    if args.op == "solve":
        run_solve(args, world, rank, local)
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
