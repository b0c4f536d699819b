mkdir -p gpurun_out
for v in "" "VSP_NO_MULTICAST=1" "VSP_NO_Q_PREFETCH=1"; do
  env $v timeout 300 python tools/k3_trace.py --pattern _exp_data/pat.pt > /dev/null 2>> gpurun_out/k3_trace.err
  python - "$v" <<'PY'
import numpy as np, sys
ev=np.load('gpurun_out/k3_trace_sparse.npy').astype(np.int64)
per=ev[0,0,1:]-ev[0,0,:-1]
idx=np.where(per>4500)[0]
q=[ev[7,1,G+1]-ev[7,0,G+1] for G in idx]
print(sys.argv[1] or 'default', 'median period', np.median(per), 'boundaries', len(idx), 'median boundary', np.median(per[idx]) if len(idx) else 0, 'Q load clk median', np.median(q) if q else 0, 'total clk', ev[0,0,-1]-ev[0,0,0])
PY
done
