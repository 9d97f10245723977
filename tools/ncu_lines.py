"""Rank CUDA source lines of one kernel in an .ncu-rep by executed warp instructions.

    python tools/ncu_lines.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, out = None, None, []
    for r in csv.reader(io.StringIO(txt)):
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[0] == "":
            continue
        try:
            out.append((int(r[7]), int(r[4]), cur, r[0], r[1][:100]))
        except ValueError:
            pass
    out.sort(reverse=True)
    print("total warp instructions", sum(o[0] for o in out), "stall samples", sum(o[1] for o in out))
    for o in out[:n]:
        print(f"{o[0]:10d} {o[1]:6d} {o[2]}:{o[3]} {o[4]}")


if __name__ == "__main__":
    main()
