set -x
nproc; grep -m1 "model name" /proc/cpuinfo; nvidia-smi --query-gpu=name,clocks.sm,power.limit --format=csv
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/pytest_gpu.txt 2>&1
tail -25 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
tail -c 1500 gpurun_out/ref.json
