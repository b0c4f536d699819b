# §8f kernels at the headline geometry: timings + rooflines, then ncu DRAM bytes of the RoPE launches
mkdir -p gpurun_out
timeout 600 python tools/f_rows_bench.py > gpurun_out/f_rows.jsonl 2> gpurun_out/f_rows.err; cat gpurun_out/f_rows.jsonl; tail -3 gpurun_out/f_rows.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"rope|recall|kl_grad|backward|adamw|indexer_gemm" -c 40 --csv --log-file gpurun_out/f_rows_ncu.csv python tools/f_rows_bench.py > /dev/null 2>&1
python - <<'PY'
import csv,collections,statistics
rows=list(csv.reader(open('gpurun_out/f_rows_ncu.csv')))
h=[i for i,x in enumerate(rows) if 'Kernel Name' in x][0]; H=rows[h]
ik,im,iv=H.index('Kernel Name'),H.index('Metric Name'),H.index('Metric Value')
d=collections.defaultdict(lambda: collections.defaultdict(list))
for x in rows[h+1:]: d[x[ik][:60]][x[im]].append(float(x[iv].replace(',','')))
for k,m in d.items(): print(k, {a:round(statistics.median(b),1) for a,b in m.items()})
PY
