mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches.csv python tools/bench_configs.py c1 > gpurun_out/c1_ncu.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c1_launches.csv')))
h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
hdr=rows[h]; ik=hdr.index('Kernel Name'); iv=hdr.index('Metric Value')
from collections import defaultdict
d=defaultdict(list)
for r in rows[h+1:]: d[r[ik][:70]].append(float(r[iv].replace(',',''))/1e3)
for k,v in d.items(): print(f"{k:70s} n={len(v)} min={min(v):.1f} med={sorted(v)[len(v)//2]:.1f} us")
PY
