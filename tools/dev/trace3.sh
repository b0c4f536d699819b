for v in "" "VSP_DEBUG_NO_O_STORE=1"; do
  env $v timeout 300 python tools/k3_trace.py --pattern _exp_data/pat.pt > /dev/null 2>> gpurun_out/k3_trace.err
  python - "$v" <<'PY'
import numpy as np, sys
ev=np.load('gpurun_out/k3_trace_sparse.npy').astype(np.int64)
per=ev[0,0,1:]-ev[0,0,:-1]
idx=np.where(per>4500)[0]
print(sys.argv[1] or 'default', 'median period', np.median(per), 'boundaries', len(idx), 'median boundary', np.median(per[idx]) if len(idx) else 0, 'sum boundary excess', (per[idx]-np.median(per)).sum(), 'total', per[per>0].sum())
PY
done
