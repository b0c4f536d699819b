mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_config_parity.py tests/test_gpu_attention.py tests/test_gpu_fullsize.py tests/test_gpu_sharding.py -x -q > gpurun_out/c1_tests.txt 2>&1; tail -15 gpurun_out/c1_tests.txt
timeout 300 python tools/bench_configs.py c1 c2 > gpurun_out/c1_cfg.jsonl 2>&1; cat gpurun_out/c1_cfg.jsonl
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
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_quick.json 2>gpurun_out/bench_quick.err; head -c 400 gpurun_out/bench_quick.json; grep -o '"roofline.*"kernel_ms": [0-9.]*' gpurun_out/bench_quick.json
