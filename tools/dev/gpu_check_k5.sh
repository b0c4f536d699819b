set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/gpu_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:aggregate_kernel -c 1 -o gpurun_out/prof_k5_32k python tools/prof_driver.py --what aggregate --iters 1 > gpurun_out/prof_k5.log 2>&1
timeout 900 ncu --section MemoryWorkloadAnalysis --section SpeedOfLight --clock-control none --nvtx --nvtx-include "timed/" -k regex:attn_fwd_kernel -c 2 -o gpurun_out/prof_k3_traffic python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_k3t.log 2>&1
tail -3 gpurun_out/gpu_tests.log
