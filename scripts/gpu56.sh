cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches56.csv python bench.py --config delicious_als > gpurun_out/bench56.json 2>&1
python3 - <<'PY'
import csv
from collections import defaultdict
rows=list(csv.reader(open("gpurun_out/launches56.csv")))
st=next(i for i,r in enumerate(rows) if r and r[0]=="ID")
h=rows[st]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
agg=defaultdict(list)
for r in rows[st+1:]:
    if len(r)>vi: agg[r[ki].split("(")[0][-40:]].append(float(r[vi]))
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1])):
    print(f"{k:42s} n={len(v):4d} total={sum(v)/1e6:8.2f} ms  min={min(v)/1e3:9.1f} us max={max(v)/1e3:9.1f} us")
PY
