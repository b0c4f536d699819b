export VSP_ATTN_1H=1
timeout 300 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fullsize.py tests/test_gpu_config_parity.py -x -q 2>&1 | tail -4
unset VSP_ATTN_1H
for r in 1 2; do
  for v in 0 1; do
  VSP_ATTN_1H=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/h$v.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/h$v.json').read().strip().splitlines()[-1])
print('1h=$v', round(b['ms_per_step'],3), 'k3', round(b['roofline']['kernel_ms'],3), 'dense', round(b['dense_ms'],2), 'recall', b['recall'], b['clocks']['sm_mhz'], b['clocks']['reasons'])"
  done
done
