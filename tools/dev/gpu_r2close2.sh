set -x
mkdir -p gpurun_out/close2
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/close2/pytest_gpu.txt 2>&1; tail -2 gpurun_out/close2/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python tools/bench_configs.py c1 c2 > gpurun_out/close2/configs_c12.jsonl 2> gpurun_out/close2/configs.err; cut -c1-600 gpurun_out/close2/configs_c12.jsonl; tail -2 gpurun_out/close2/configs.err
