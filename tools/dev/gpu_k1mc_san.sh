# K1 W_U multicast clusters: repeated bit-identity test + memcheck / synccheck / racecheck on it
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for i in 1 2 3 4 5; do timeout 300 python -m pytest tests/test_gpu_indexer_select.py -q -k multicast 2>&1 | tail -1; done
for tool in memcheck synccheck racecheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 9 python -m pytest tests/test_gpu_indexer_select.py -q -x -k "multicast and not 131072" > gpurun_out/san_k1mc_$tool.log 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/san_k1mc_$tool.log
done
