# one ncu --set full capture of the transposed distillation backward (f_rows_bench distill leg)
mkdir -p gpurun_out/bwd
timeout 900 ncu --set full --import-source on --clock-control none -k regex:backward_kernel -s 2 -c 1 -o gpurun_out/bwd/bwd python tools/f_rows_bench.py > gpurun_out/bwd/ncu.log 2>&1; tail -2 gpurun_out/bwd/ncu.log
ncu -i gpurun_out/bwd/bwd.ncu-rep --page raw --csv > gpurun_out/bwd/raw.csv 2>/dev/null
ncu -i gpurun_out/bwd/bwd.ncu-rep --page details --csv > gpurun_out/bwd/details.csv 2>/dev/null
ls -la gpurun_out/bwd
