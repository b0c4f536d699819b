# kernel-level ncu durations for several package builds on the bench layer:
#   bash tools/dev/gpu_ab_dirs.sh <kernel regex> dir1 dir2 ...
K=$1; shift
mkdir -p gpurun_out
for r in 1 2; do for d in "$@"; do
  VSP_ROOT=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$K --csv --log-file gpurun_out/abd.csv python tools/dev/layer_run.py > /dev/null 2>&1
  python -c "
import csv,statistics
rows=list(csv.reader(open('gpurun_out/abd.csv')))
h=[i for i,x in enumerate(rows) if 'Kernel Name' in x][0]; iv=rows[h].index('Metric Value')
t=[float(x[iv].replace(',',''))/1e3 for x in rows[h+1:]]
print('$d $K us: median %.1f min %.1f n=%d' % (statistics.median(t), min(t), len(t)))"
done; done
