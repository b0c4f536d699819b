./tools/dev/tofix_check
timeout 600 python -m pytest tests/test_gpu_indexer_select.py tests/test_gpu_misc_ops.py tests/test_gpu_config_parity.py -x -q 2>&1 | tail -2
K2_CLUSTER=4 timeout 300 python tools/k2_trace.py
