"""Collapse a compute-sanitizer racecheck log (--racecheck-report hazard) into unique
(kind, write site, read site) triples with counts."""
import collections
import re
import sys

pairs = collections.Counter()
cur = None
for line in open(sys.argv[1], errors="replace"):
    m = re.search(r"Error: Potential (\w+) hazard", line)
    if m:
        cur = [m.group(1), "", ""]
        continue
    if cur is None:
        continue
    m = re.search(r"(Write|Read) Thread \(\d+,\d+,\d+\) at (.*?)\+0x[0-9a-f]+( in (\S+))?", line)
    if m:
        site = (m.group(2).split("(")[0][-60:] + " " + (m.group(4) or "")).strip()
        cur[1 if m.group(1) == "Write" else 2] = site
        if cur[1] and cur[2]:
            pairs[tuple(cur)] += 1
            cur = None
for (k, w, r), c in pairs.most_common():
    print(f"{c:8d} {k}  W: {w}  R: {r}")
