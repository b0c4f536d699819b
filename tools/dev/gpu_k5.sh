mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_aggregate.py tests/test_gpu_train.py -x -q 2>&1 | tail -3
for n in 32768 65536; do VSP_ROOT=_exp_base timeout 300 python tools/k5_time.py $n | sed 's/^/base /'; timeout 300 python tools/k5_time.py $n | sed 's/^/new  /'; done
