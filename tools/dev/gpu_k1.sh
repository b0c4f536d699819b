mkdir -p gpurun_out
for r in base new; do
  if [ $r = base ]; then export VSP_ROOT=_exp_base; else unset VSP_ROOT; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:indexer_gemm --csv --log-file gpurun_out/k1_$r.csv python tools/dev/k1_time.py > /dev/null 2>&1
  python -c "
import csv,statistics
rows=list(csv.reader(open('gpurun_out/k1_$r.csv')))
h=[i for i,x in enumerate(rows) if 'Kernel Name' in x][0]; iv=rows[h].index('Metric Value')
t=[float(x[iv].replace(',',''))/1e3 for x in rows[h+1:]]
print('$r indexer_gemm us: median %.1f min %.1f n=%d' % (statistics.median(t), min(t), len(t)))"
done
unset VSP_ROOT
timeout 600 python -m pytest tests/test_gpu_indexer_select.py tests/test_gpu_config_parity.py -q -x 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none -k regex:indexer_gemm -c 1 -o gpurun_out/prof_k1 python tools/dev/k1_time.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_k1.ncu-rep 2>&1 | head -22
