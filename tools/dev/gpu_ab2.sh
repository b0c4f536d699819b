# 20-step bench A/B of _exp_base vs _exp_new (alternating), K3 live time and the dense K4 time
for r in 1 2 3; do for v in base new; do
  VSP_ROOT=_exp_$v timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab2_$v.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/ab2_$v.json').read().strip().splitlines()[-1])
print('$v', round(b['ms_per_step'],3), 'k3', round(b['roofline']['kernel_ms'],3), 'dense', round(b['dense_ms'],2), b['clocks']['sm_mhz'], b['clocks']['reasons'])"
done; done
