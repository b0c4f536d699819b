# A/B of the attention kernels: _exp_base (previous build) vs the working tree, alternating
# processes on the same bench layer and pattern. Usage: bash tools/dev/ab.sh [reps]

mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
R=${1:-3}
timeout 400 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fullsize.py tests/test_gpu_config_parity.py -x -q > gpurun_out/ab_tests.txt 2>&1; tail -3 gpurun_out/ab_tests.txt
mkdir -p _exp_data; [ -f _exp_data/pat.pt ] || timeout 300 python tools/k3_ab.py --pattern _exp_data/pat.pt --reps 3 > /dev/null 2>&1; cp _exp_data/pat.pt gpurun_out/pat.pt
for i in $(seq $R); do
  VSP_ROOT=_exp_base timeout 120 python tools/k3_ab.py --layer 1 --reps 20 2>/dev/null | sed 's/^/base layer  /' | tee -a gpurun_out/ab.txt
  timeout 120 python tools/k3_ab.py --layer 1 --reps 20 2>/dev/null | sed 's/^/new  layer  /' | tee -a gpurun_out/ab.txt
  VSP_ROOT=_exp_base timeout 120 python tools/k3_ab.py --pattern _exp_data/pat.pt --reps 20 2>/dev/null | sed 's/^/base sparse /' | tee -a gpurun_out/ab.txt
  timeout 120 python tools/k3_ab.py --pattern _exp_data/pat.pt --reps 20 2>/dev/null | sed 's/^/new  sparse /' | tee -a gpurun_out/ab.txt
  VSP_ROOT=_exp_base timeout 120 python tools/k3_ab.py --pattern _exp_data/pat.pt --reps 3 --dense 1 2>/dev/null | sed 's/^/base dense /' | tee -a gpurun_out/ab.txt
  timeout 120 python tools/k3_ab.py --pattern _exp_data/pat.pt --reps 3 --dense 1 2>/dev/null | sed 's/^/new  dense /' | tee -a gpurun_out/ab.txt
done
