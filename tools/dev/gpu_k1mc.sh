# K1 W_U multicast cluster size A/B (VSP_K1_MC = 1 / 2 / 4): parity, then kernel time under ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_indexer_select.py -q -x 2>&1 | tail -3
for mc in 1 2 4 1 2 4; do
  VSP_K1_MC=$mc timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum --clock-control none -k regex:indexer_gemm --csv --log-file gpurun_out/k1mc_$mc.csv python tools/dev/k1_time.py > /dev/null 2>&1
  python - <<PY
import csv,statistics
rows=list(csv.reader(open('gpurun_out/k1mc_$mc.csv')))
h=[i for i,x in enumerate(rows) if 'Kernel Name' in x][0]; iv=rows[h].index('Metric Value'); im=rows[h].index('Metric Name')
d={}
for x in rows[h+1:]: d.setdefault(x[im],[]).append(float(x[iv].replace(',','')))
print('mc=$mc', {k:round(statistics.median(v),1) for k,v in d.items()})
PY
  VSP_K1_MC=$mc python tools/dev/k1_time.py
done
