"""Rank CUDA source lines of the first kernel in an .ncu-rep by stall samples.

    python tools/ncu_hot.py report.ncu-rep [N] [kernel-substring]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
sub = sys.argv[3] if len(sys.argv) > 3 else ""
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = hdr = fn = None
out = []
for r in csv.reader(io.StringIO(txt)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Function Name":
        fn = r[1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "" or (sub and sub not in (fn or "")):
        continue
    try:
        out.append((int(r[4]), int(r[7]), cur, r[0], r[1][:96]))
    except ValueError:
        pass
print("stall samples", sum(o[0] for o in out), "warp instructions", sum(o[1] for o in out))
for o in sorted(out, reverse=True)[:n]:
    print(f"{o[0]:7d} {o[1]:10d} {o[2]}:{o[3]} {o[4]}")
