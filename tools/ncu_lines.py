"""Per-source-line warp-stall samples of an ncu report (cuda,sass source view): the top lines
and the totals per named kernel region.  Usage: python tools/ncu_lines.py REPORT [top]"""
import csv
import collections
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
per_line = collections.Counter()
per_stall = collections.defaultdict(collections.Counter)
src_text = {}
fname = None
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < len(hdr) or not r[0].isdigit():
        continue
    # the cuda-level rows carry line number + source; sass rows repeat with an address
    d = dict(zip(hdr[2:], r[2:]))
    if r[2] != "-":  # an address: a SASS row (its samples are in the enclosing cuda line)
        continue
    try:
        n = int(float(d.get("Warp Stall Sampling (All Samples)", "0") or 0))
    except ValueError:
        continue
    key = (fname, int(r[0]))
    per_line[key] += n
    src_text[key] = r[1].strip()[:90]
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                per_stall[key][k[6:]] += int(float(v or 0))
            except ValueError:
                pass
tot = sum(per_line.values()) or 1
print(f"total samples {tot}")
for key, n in per_line.most_common(top):
    st = ", ".join(f"{k} {v}" for k, v in per_stall[key].most_common(3) if v)
    print(f"{100 * n / tot:5.1f}% {key[0]}:{key[1]:<5} {src_text[key]:<90} [{st}]")
