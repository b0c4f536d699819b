export VSP_ATTN_1H=1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:attn1h -c 1 -o gpurun_out/prof_1h python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_1h.log 2>&1
ls gpurun_out/prof_1h*
