# K1 W_U ring depth A/B: 4 stages (tree) vs 5 stages (d_h <= 1024 staging), kernel time under ncu
mkdir -p gpurun_out
for d in tree _exp_s5 tree _exp_s5; do
  if [ $d = tree ]; then unset VSP_ROOT; else export VSP_ROOT=$d; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:indexer_gemm --csv --log-file gpurun_out/k1s_$d.csv python tools/dev/k1_time.py > /dev/null 2>&1
  python - <<PY
import csv,statistics
rows=list(csv.reader(open('gpurun_out/k1s_$d.csv')))
h=[i for i,x in enumerate(rows) if 'Kernel Name' in x][0]; iv=rows[h].index('Metric Value')
t=[float(x[iv].replace(',',''))/1e3 for x in rows[h+1:]]
print('$d indexer_gemm us: median %.1f min %.1f n=%d' % (statistics.median(t), min(t), len(t)))
PY
done
unset VSP_ROOT
