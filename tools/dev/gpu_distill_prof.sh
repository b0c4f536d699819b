# per-kernel breakdown of one distillation step (f_rows_bench distill leg) at 128k x 8 heads
mkdir -p gpurun_out/distill
timeout 600 ncu --metrics gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"kl_grad|backward|adamw|indexer_gemm|reduce_grads|sum_loss" -c 60 --csv --log-file gpurun_out/distill/ncu.csv python tools/f_rows_bench.py > gpurun_out/distill/out.log 2>&1
python - <<'PY'
import csv,collections,statistics
rows=list(csv.reader(open('gpurun_out/distill/ncu.csv')))
h=[i for i,x in enumerate(rows) if 'Kernel Name' in x][0]; H=rows[h]
ik,im,iv=H.index('Kernel Name'),H.index('Metric Name'),H.index('Metric Value')
ig=H.index('Grid Size') if 'Grid Size' in H else None
d=collections.defaultdict(lambda: collections.defaultdict(list))
for x in rows[h+1:]: d[x[ik][:70]+(' '+x[ig] if ig else '')][x[im]].append(float(x[iv].replace(',','')))
for k,m in d.items(): print(k, {a:round(statistics.median(b),1) for a,b in m.items()}, 'count', len(next(iter(m.values()))))
PY
