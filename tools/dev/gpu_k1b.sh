bash tools/dev/gpu_ab_kernel.sh indexer_gemm
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
