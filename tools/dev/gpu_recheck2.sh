# GPU suite, smoke, default bench, 20-step bench, and a 20-step bench with the previous K1 layout
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench20.json 2> gpurun_out/bench20.err
VSP_K1_SPLIT=0 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench20_nosplit.json 2>/dev/null
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench20_b.json 2>/dev/null
python - <<'PY'
import json
for f in ['bench','bench20','bench20_nosplit','bench20_b']:
    try:
        d=json.load(open('gpurun_out/%s.json'%f))
        print(f, round(d['value']/1e6,2), 'Mtok/s', round(d['ms_per_step'],3), 'ms/step K3 frac', round(d['roofline']['frac'],3), 'k1', round(d['indexer_ms'],3), 'e2e', round(d['e2e']['value']/1e6,2), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
    except Exception as e: print(f, 'ERR', e)
PY
