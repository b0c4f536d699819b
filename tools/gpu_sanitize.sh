# compute-sanitizer over the CUDA path on one B200: memcheck (smoke + the GPU parity suite at
# small sizes), synccheck and racecheck (smoke). Logs under gpurun_out/.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_memcheck_smoke.log 2>&1; echo MEMCHECK_SMOKE=$? >> gpurun_out/san_memcheck_smoke.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_attention.py tests/test_gpu_indexer_select.py tests/test_gpu_aggregate.py tests/test_gpu_train.py tests/test_gpu_rope.py tests/test_gpu_sharding.py -x -q -k "not long and not 131072 and not 300001" > gpurun_out/san_memcheck_tests.log 2>&1; echo MEMCHECK_TESTS=$? >> gpurun_out/san_memcheck_tests.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_synccheck_smoke.log 2>&1; echo SYNCCHECK=$? >> gpurun_out/san_synccheck_smoke.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_racecheck_smoke.log 2>&1; echo RACECHECK=$? >> gpurun_out/san_racecheck_smoke.log
for f in gpurun_out/san_*.log; do echo "== $f"; tail -3 $f; done
