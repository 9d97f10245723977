# per-kernel device times of one msed_dual / tape call at c3 UpGate (ncu launch list, cold caches)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/prof_tc.py 2>/dev/null | grep -v "^==" > gpurun_out/launches_tc.csv
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches_tc.csv')))
rows=[r for r in rows if len(r)>5]; h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value"); ii=h.index("ID")
from collections import defaultdict
d=defaultdict(dict); names={}
for r in rows[1:]:
    d[r[ii]][r[mi]]=r[vi]; names[r[ii]]=r[ki][:70]
for i in sorted(d, key=int):
    m=d[i]; print(i, names[i], m.get("gpu__time_duration.sum"), "ns  R", m.get("dram__bytes_read.sum"), "W", m.get("dram__bytes_write.sum"))
PY
