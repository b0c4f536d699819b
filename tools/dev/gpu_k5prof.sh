# K5 counters of _exp_* builds vs the working tree at a given n (default 65536)
N=${1:-65536}
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size
mkdir -p gpurun_out
for d in _exp_* tree; do
  if [ $d = tree ]; then unset VSP_ROOT; else export VSP_ROOT=$d; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:aggregate_kernel -c 1 --csv --log-file gpurun_out/k5prof_$d.csv python tools/k5_time.py $N > /dev/null 2>&1
  python -c "
import csv
rows=list(csv.reader(open('gpurun_out/k5prof_$d.csv')))
h=[i for i,r in enumerate(rows) if 'Metric Name' in r][0]
iN=rows[h].index('Metric Name'); iV=rows[h].index('Metric Value')
print('$d', ' '.join('%s=%s'%(r[iN], r[iV]) for r in rows[h+1:]))"
done
