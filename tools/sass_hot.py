"""Per-SASS-instruction hot spots of one kernel in an .ncu-rep: totals, opcode mix,
and the top instructions by stall samples.

    python tools/sass_hot.py report.ncu-rep kernel-regex [launch-skip] [N]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      "regex:" + kre, "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
recs = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    recs.append((r[ix["Address"]], r[ix["Source"]].strip(), int(r[ix["Warp Stall Sampling (All Samples)"]]),
                 int(r[ix["Instructions Executed"]]), int(r[ix["Thread Instructions Executed"]])))
tot_s = sum(r[2] for r in recs)
tot_i = sum(r[3] for r in recs)
tot_t = sum(r[4] for r in recs)
print(f"{rows[0][1][:90]}: samples {tot_s}  warp-inst {tot_i}  thread-inst {tot_t}")
ops = collections.Counter()
for r in recs:
    ops[r[1].split()[0] if not r[1].startswith("@") else r[1].split()[1]] += r[3]
print("opcode mix (warp instructions):")
for op, c in ops.most_common(30):
    print(f"  {op:22s} {c:12d} {c / tot_i:6.1%}")
print("top by samples:")
for i, r in sorted(enumerate(recs), key=lambda x: -x[1][2])[:n]:
    print(f"{i:6d} {r[2]:7d} {r[3]:10d}  {r[1][:90]}")
if len(sys.argv) > 5:
    with open(sys.argv[5], "w") as f:
        half = len(recs)
        for i, r in enumerate(recs):
            f.write(f"{i:6d} {r[2]:6d} {r[3]:10d}  {r[1]}\n")
