# K1 with and without its epilogue math (build the probe first:
#   python tools/dev/build_variant.py _exp_noepi -DVSP_K1_NOEPI)
for d in _exp_noepi tree; do
  if [ $d = tree ]; then unset VSP_ROOT; else export VSP_ROOT=$d; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:indexer_gemm -c 1 python tools/dev/k1_time.py 2>&1 | grep -E "duration|tensor|lts__" | sed "s/^/$d /"
done
