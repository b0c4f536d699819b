# K5 variants: parity of the working tree, then pass-2 timings of every _exp_* build vs the tree
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_aggregate.py -x -q 2>&1 | tail -3
for n in 32768 65536; do
  for r in 1 2; do
    for d in _exp_*; do VSP_ROOT=$d timeout 300 python tools/k5_time.py $n | sed "s/^/$d /"; done
    timeout 300 python tools/k5_time.py $n | sed 's/^/tree /'
  done
done
