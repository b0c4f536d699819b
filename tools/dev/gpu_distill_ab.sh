# distillation step after the train.cu changes: parity tests, timing, per-kernel ncu breakdown
mkdir -p gpurun_out/distill5
timeout 300 python -m pytest tests/test_gpu_train.py -q -x > gpurun_out/distill5/pytest.txt 2>&1; tail -3 gpurun_out/distill5/pytest.txt
timeout 600 python tools/f_rows_bench.py > gpurun_out/distill5/f_rows.jsonl 2> gpurun_out/distill5/f_rows.err; grep distill gpurun_out/distill5/f_rows.jsonl | cut -c1-400; tail -3 gpurun_out/distill5/f_rows.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"kl_grad|backward|adamw|indexer_gemm|reduce_grads|sum_loss" -c 60 --csv --log-file gpurun_out/distill5/ncu.csv python tools/f_rows_bench.py > /dev/null 2>&1
python - <<'PY'
import csv,collections,statistics
rows=list(csv.reader(open('gpurun_out/distill5/ncu.csv')))
h=[i for i,x in enumerate(rows) if 'Kernel Name' in x][0]; H=rows[h]
ik,im,iv,ig=H.index('Kernel Name'),H.index('Metric Name'),H.index('Metric Value'),H.index('Grid Size')
d=collections.defaultdict(list)
for x in rows[h+1:]:
    try: d[x[ik][:50]+' '+x[ig]].append(float(x[iv].replace(',','')))
    except: pass
for k,m in d.items(): print(k, round(statistics.median(m)/1e3,1),'us n',len(m))
PY
