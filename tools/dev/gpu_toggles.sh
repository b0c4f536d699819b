for r in 1 2; do for t in none VSP_NO_Q_PREFETCH VSP_NO_MULTICAST; do
  if [ $t = none ]; then E=""; else E="$t=1"; fi
  env $E timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/tg.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/tg.json').read().strip().splitlines()[-1])
print('$t', round(b['ms_per_step'],3), 'k3', round(b['roofline']['kernel_ms'],3), b['clocks']['sm_mhz'], b['clocks']['reasons'])"
done; done
