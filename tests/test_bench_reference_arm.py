"""bench.py --impl reference on CPU: the reference's own assembly (oracle/_ref) on config 1 at its
full size, one JSON line with the arm's contract keys, and the repo's CUDA library never loaded
in that process (the reference arm must not run any of our code)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_and_no_repo_library():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libdgref.so")):
        pytest.skip("oracle/_ref (the compiled reference) is not built")
    code = (
        "import runpy, sys\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', '--config', '1']\n"
        "runpy.run_path('bench.py', run_name='__main__')\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('REPO_SO_LOADED' if 'libdgfem_b200' in maps else 'REPO_SO_NOT_LOADED')\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert lines[-1] == "REPO_SO_NOT_LOADED"
    d = json.loads(lines[-2])
    assert d["impl"] == "reference" and d["unit"] == "elements/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("config 1: 32x32")
    assert "= the full config" in d["sample"]
