"""Summarises ncu captures from gpurun_out/ into profiles/ (committed evidence).

    python tools/summarize_ncu.py [round_tag]

Reads gpurun_out/<tag>_c{1..5}.ncu-rep (ncu --set full of the block-row kernel; round 1 named
them prof_c*), gpurun_out/<tag>_spmv.ncu-rep (the BSR SpMV on config 4) and
gpurun_out/launches_<tag>_c<L>.csv (per-launch gpu__time_duration list of the headline command,
L = $LAUNCH_CFG, default 4), writes profiles/ncu_summary.json (bench.py reads
dram_bytes_per_launch for roofline.traffic), profiles/ncu_<tag>_c<cfg>.txt,
profiles/ncu_<tag>_spmv.txt and profiles/launches_<tag>_c<L>.csv.
"""
from __future__ import annotations

import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.environ.get("NCU_IN", os.path.join(ROOT, "gpurun_out"))
PROF = os.environ.get("PROF_DIR", os.path.join(ROOT, "profiles"))
ELEMENTS = {1: 2048, 2: 131072, 3: 2097152, 4: 8388608, 5: 524288}

DETAILS = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active",
           "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
           "Theoretical Occupancy", "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate",
           "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block",
           "Block Size", "Grid Size", "SM Frequency"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum"]


def ncu_csv(rep: str, *args) -> list[list[str]]:
    r = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def assemblies_per_launch(cfg: int) -> int:
    """The bench line's roofline.assemblies_per_launch (dgb_assemble_batch), else 1."""
    try:
        with open(os.path.join(OUT, f"bench_c{cfg}.json")) as f:
            return int(json.load(f)["roofline"].get("assemblies_per_launch", 1) or 1)
    except Exception:
        return 1


def summarize(rep: str, cfg: int) -> dict:
    rows = ncu_csv(rep, "--page", "details")
    h = rows[0]
    det = {}
    for row in rows[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in DETAILS:
            det[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    raw = ncu_csv(rep, "--page", "raw", "--print-units", "base")
    hdr, vals = raw[0], raw[2] if len(raw) > 2 else raw[1]
    rawd = {k: v for k, v in zip(hdr, vals) if k in RAW}
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
              for k, v in zip(hdr, vals)
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and v.replace(".", "", 1).isdigit()}
    tot = sum(stalls.values()) or 1.0
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]

    def num(k):
        try:
            return float(rawd[k].replace(",", ""))
        except Exception:
            return None
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    inst = num("smsp__inst_executed.sum")
    return {
        "kernel": "block-row assembly kernel", "config": cfg,
        "details": det,
        "dram_bytes_read": rd, "dram_bytes_write": wr,
        "dram_bytes_per_launch": (rd + wr) if rd is not None and wr is not None else None,
        "assemblies_per_launch": assemblies_per_launch(cfg),
        "warp_instructions_per_element": (inst / (ELEMENTS[cfg] * assemblies_per_launch(cfg))
                                          if inst else None),
        "fp64_pipe_active_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "stall_share_pct": {k: round(100 * v / tot, 1) for k, v in top},
        "note": "ncu --set full --clock-control none (cold caches, serialised replay): use "
                "shares and traffic, not absolute time, for comparisons with bench.py",
    }


def launch_shares(path: str) -> dict:
    rows = list(csv.reader(open(path)))
    # ncu --csv log: header row containing "Kernel Name" and "Metric Value"
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    per = {}
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki]
        short = ("assemble_kernel" if "assemble_" in name else
                 "count_blocks_kernel" if "count_blocks" in name else
                 "adjacency_kernel" if "adjacency" in name else
                 "l2_flush_fill (outside the timed events)" if "FillFunctor" in name else
                 "cub_scan" if "cub" in name.lower() or "Scan" in name else name[:40])
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        per.setdefault(short, []).append(v)
    tot = sum(sum(v) for v in per.values())
    return {k: {"launches": len(v), "total_ns": sum(v), "share": round(sum(v) / tot, 4)}
            for k, v in per.items()}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    summary_path = os.path.join(PROF, "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    for cfg in (1, 2, 3, 4, 5):
        rep = os.path.join(OUT, f"{tag}_c{cfg}.ncu-rep")
        if not os.path.exists(rep):
            rep = os.path.join(OUT, f"prof_c{cfg}.ncu-rep")
        if not os.path.exists(rep):
            continue
        s = summarize(rep, cfg)
        s["round"] = tag
        summary[f"config{cfg}"] = s
        with open(os.path.join(PROF, f"ncu_{tag}_c{cfg}.txt"), "w") as f:
            f.write(json.dumps(s, indent=2) + "\n")
    rep = os.path.join(OUT, f"{tag}_spmv.ncu-rep")
    if os.path.exists(rep):
        s = summarize(rep, 4)
        s["kernel"] = "BSR SpMV (config 4 matrix)"
        s["assemblies_per_launch"] = None
        s["warp_instructions_per_row"] = s.pop("warp_instructions_per_element")
        s["round"] = tag
        summary["spmv_config4"] = s
        with open(os.path.join(PROF, f"ncu_{tag}_spmv.txt"), "w") as f:
            f.write(json.dumps(s, indent=2) + "\n")
    lcfg = int(os.environ.get("LAUNCH_CFG", "4"))
    lc = os.path.join(OUT, f"launches_{tag}_c{lcfg}.csv")
    if not os.path.exists(lc):
        lc = os.path.join(OUT, f"launches_c{lcfg}.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(PROF, f"launches_{tag}_c{lcfg}.csv"))
        summary[f"launch_shares_c{lcfg}"] = launch_shares(lc)
    with open(summary_path, "w") as f:
        json.dump(summary, f, indent=2)
    print(json.dumps({k: (v.get("dram_bytes_per_launch"), v.get("warp_instructions_per_element"),
                          v.get("details", {}).get("Duration")) if isinstance(v, dict) and "details" in v else v
                      for k, v in summary.items()}, indent=1))


if __name__ == "__main__":
    main()
