# A/B on one box: _exp_base (HEAD build) vs the working tree. Usage: bash tools/dev/gpu_ab.sh [reps]
mkdir -p gpurun_out _exp_data
R=${1:-3}
[ -f _exp_data/pat.pt ] || timeout 300 python tools/k3_ab.py --pattern _exp_data/pat.pt --reps 3 > /dev/null 2>&1
for i in $(seq $R); do
  VSP_ROOT=_exp_base timeout 120 python tools/k3_ab.py --pattern _exp_data/pat.pt --reps 20 2>/dev/null | sed 's/^/base sparse /'
  timeout 120 python tools/k3_ab.py --pattern _exp_data/pat.pt --reps 20 2>/dev/null | sed 's/^/new  sparse /'
done
PROBE_RANDOM=1 PROBE_N=4096 VSP_ROOT=_exp_base timeout 120 python tools/dev/switch_probe.py 2>&1 | tail -1 | sed 's/^/base c1like /'
PROBE_RANDOM=1 PROBE_N=4096 timeout 120 python tools/dev/switch_probe.py 2>&1 | tail -1 | sed 's/^/new  c1like /'
