mkdir -p gpurun_out
timeout 300 python tools/k3_trace.py --pattern _exp_data/pat.pt > gpurun_out/k3_trace.json 2> gpurun_out/k3_trace.err
timeout 300 python tools/k3_trace.py --pattern _exp_data/pat.pt --dense 1 >> gpurun_out/k3_trace.json 2>> gpurun_out/k3_trace.err
cat gpurun_out/k3_trace.json; tail -3 gpurun_out/k3_trace.err
