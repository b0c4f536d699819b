for r in 1 2; do for v in p6 p0 p4 p8; do
  VSP_ROOT=_exp_$v timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/poly_$v.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/poly_$v.json').read().strip().splitlines()[-1])
print('$v', round(b['ms_per_step'],3), 'k3', round(b['roofline']['kernel_ms'],3), b['clocks']['sm_mhz'], b['clocks']['reasons'])"
done; done
