# K1 split-X layout (VSP_K1_SPLIT=1) vs default: bit identity (incl. d_h = 256 single-chunk items), ncu time
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_indexer_select.py -q -x -k "pairs" 2>&1 | tail -2
VSP_K1_SPLIT=1 timeout 300 python -m pytest tests/test_gpu_indexer_select.py -q -x 2>&1 | tail -2
for rep in 1 2; do
for sp in 0 1; do
  VSP_K1_SPLIT=$sp timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:indexer_gemm --csv --log-file gpurun_out/k1s_$sp.csv python tools/dev/k1_time.py > /dev/null 2>&1
  python - <<PY
import csv,statistics,collections
rows=list(csv.reader(open('gpurun_out/k1s_$sp.csv')))
h=[i for i,x in enumerate(rows) if 'Kernel Name' in x][0]; H=rows[h]; im,iv=H.index('Metric Name'),H.index('Metric Value')
d=collections.defaultdict(list)
for x in rows[h+1:]: d[x[im]].append(float(x[iv].replace(',','')))
print('split=$sp', {k:round(statistics.median(v),1) for k,v in d.items()})
PY
  VSP_K1_SPLIT=$sp timeout 120 python tools/dev/k1_time.py
done
done
