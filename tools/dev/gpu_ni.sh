for r in 1 2; do for v in base ni; do
  VSP_ROOT=_exp_$v timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ni_$v.json 2>/dev/null
  python -c "
import json; b=json.loads(open('gpurun_out/ni_$v.json').read().strip().splitlines()[-1])
print('$v', round(b['ms_per_step'],3), 'k3', round(b['roofline']['kernel_ms'],3), b['clocks']['sm_mhz'], b['clocks']['reasons'])"
  PROBE_RANDOM=1 PROBE_N=4096 VSP_ROOT=_exp_$v timeout 120 python tools/dev/switch_probe.py 2>&1 | tail -1 | sed "s/^/$v c1like /"
done; done
