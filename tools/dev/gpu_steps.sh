for s in 5 20 50 5; do
  timeout 600 python bench.py --steps $s --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/steps_$s.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/steps_$s.json').read().strip().splitlines()[-1])
print('steps=$s', round(b['ms_per_step'],3), 'k3', round(b['roofline']['kernel_ms'],3), 'idx', round(b['indexer_ms']*1e3,1), b['clocks'])"
done
nvidia-smi --query-gpu=power.draw,power.limit,temperature.gpu,clocks.sm,clocks_throttle_reasons.active --format=csv
