set -x
nproc; free -g | head -2; grep -m1 "model name" /proc/cpuinfo; nvidia-smi --query-gpu=name,clocks.sm,power.limit --format=csv
mkdir -p gpurun_out
timeout 900 python bench.py --prep fresh --save-prep --steps 5 --warmup 3 > gpurun_out/bench_prep.json 2> gpurun_out/bench_prep.err
cp -r bench_data gpurun_out/ 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
tail -c 600 gpurun_out/ref.json
