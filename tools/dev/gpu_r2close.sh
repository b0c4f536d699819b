set -x
mkdir -p gpurun_out/close3
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/close3/pytest_gpu.txt 2>&1; tail -2 gpurun_out/close3/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/close3/bench.json 2> gpurun_out/close3/bench.err
head -c 400 gpurun_out/close3/bench.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/close3/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/close3/launch_bench.log 2>&1
ls gpurun_out/close3
