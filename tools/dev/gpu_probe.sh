mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_config_parity.py tests/test_gpu_attention.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
timeout 300 python tools/bench_configs.py c1 2>&1 | tail -1
timeout 300 python tools/dev/switch_probe.py 2>&1 | tail -3
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_quick.json 2>gpurun_out/bench_quick.err; head -c 300 gpurun_out/bench_quick.json; grep -o '"frac": [0-9.]*\|"kernel_ms": [0-9.]*' gpurun_out/bench_quick.json
