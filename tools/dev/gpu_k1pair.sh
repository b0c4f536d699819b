# K1 modes: one CTA / CTA pair (cta_group::2) x W_U stage of 32 / 64 K-rows: parity + bit identity, ncu time
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_indexer_select.py -q -x -k "pairs" 2>&1 | tail -2
for rep in 1 2; do
for cfg in 1_32 1_64 2_32 2_64; do
  mc=${cfg%_*}; sk=${cfg#*_}
  VSP_K1_MC=$mc VSP_K1_STAGEK=$sk timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:indexer_gemm --csv --log-file gpurun_out/k1m_$cfg.csv python tools/dev/k1_time.py > /dev/null 2>&1
  python - <<PY
import csv,statistics,collections
rows=list(csv.reader(open('gpurun_out/k1m_$cfg.csv')))
h=[i for i,x in enumerate(rows) if 'Kernel Name' in x][0]; H=rows[h]; im,iv=H.index('Metric Name'),H.index('Metric Value')
d=collections.defaultdict(list)
for x in rows[h+1:]: d[x[im]].append(float(x[iv].replace(',','')))
print('mc,stageK=$cfg', {k:round(statistics.median(v),1) for k,v in d.items()})
PY
done
done
