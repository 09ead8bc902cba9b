# usage: bash tools/ncu_lib.sh <lib.so> <mode> : key ncu metrics for one launch of that build
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,gpc__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -s 2 -c 1 --clock-control none --csv env LIBS=x=$1 MODES=$2 ROUNDS=1 REPS=1 python tools/ab_libs.py 2>/dev/null | python -c "
import csv,sys,json
rows=[r for r in csv.reader(sys.stdin) if len(r)>14 and r[0]!='ID']
d={r[12]: r[14] for r in rows}
print(sys.argv[1], sys.argv[2], 'us', round(float(d['gpu__time_duration.sum'])/1000,1), 'GHz', round(float(d['gpc__cycles_elapsed.avg.per_second'])/1e9,3), 'tensor%', d['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'], 'dramR GB', round(float(d['dram__bytes_read.sum'])/1e9,2))" $1 $2
