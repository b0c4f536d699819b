# kernel-level A/B (ncu durations) of _exp_base vs the working tree on the bench layer
# usage: bash tools/dev/gpu_ab_kernel.sh <kernel regex>
K=${1:-select_kernel}
mkdir -p gpurun_out
for r in base new base new; do
  if [ $r = base ]; then export VSP_ROOT=_exp_base; else unset VSP_ROOT; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$K --csv --log-file gpurun_out/ab_$r.csv python tools/dev/layer_run.py > /dev/null 2>&1
  python -c "
import csv,statistics
rows=list(csv.reader(open('gpurun_out/ab_$r.csv')))
h=[i for i,x in enumerate(rows) if 'Kernel Name' in x][0]; iv=rows[h].index('Metric Value')
t=[float(x[iv].replace(',',''))/1e3 for x in rows[h+1:]]
print('$r $K us: median %.1f min %.1f n=%d' % (statistics.median(t), min(t), len(t)))"
done
