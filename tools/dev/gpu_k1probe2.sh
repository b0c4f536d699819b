# K1 bound probe: full kernel / epilogue off / half the MMAs (same W and X streams) / both
mkdir -p gpurun_out
for d in tree _exp_noepi _exp_half _exp_noepi_half tree _exp_noepi _exp_half _exp_noepi_half; do
  if [ $d = tree ]; then unset VSP_ROOT; else export VSP_ROOT=$d; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:indexer_gemm --csv --log-file gpurun_out/k1p_$d.csv python tools/dev/k1_time.py > /dev/null 2>&1
  python - <<PY
import csv,statistics,collections
rows=list(csv.reader(open('gpurun_out/k1p_$d.csv')))
h=[i for i,x in enumerate(rows) if 'Kernel Name' in x][0]; H=rows[h]; im,iv=H.index('Metric Name'),H.index('Metric Value')
d=collections.defaultdict(list)
for x in rows[h+1:]: d[x[im]].append(float(x[iv].replace(',','')))
print('$d', {k:round(statistics.median(v),1) for k,v in d.items()})
PY
done
unset VSP_ROOT
