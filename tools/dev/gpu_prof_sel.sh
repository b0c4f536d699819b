mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:select_kernel -c 1 -o gpurun_out/prof_k2_bench python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_k2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_kernel -c 1 -o gpurun_out/prof_k2_c1 python tools/dev/c1_pair.py > gpurun_out/prof_k2c1.log 2>&1
ls gpurun_out/*.ncu-rep
