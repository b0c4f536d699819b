set -x
mkdir -p gpurun_out
timeout 900 python tools/bench_configs.py c1 c2 c5 > gpurun_out/configs_c125.jsonl 2> gpurun_out/configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:attn_fwd_kernel -c 1 -o gpurun_out/prof_k3_bench python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_k3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:"indexer|select|plan|gather" -c 6 -o gpurun_out/prof_small_bench python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/prof_small.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -c 1 -o gpurun_out/prof_k4_32k python tools/prof_driver.py --what dense --iters 1 > gpurun_out/prof_k4.log 2>&1
timeout 1500 python tools/bench_configs.py c4 > gpurun_out/configs_c4.jsonl 2> gpurun_out/configs_c4.err
ls gpurun_out
