# usage: bash tools/ncu_metrics.sh '<json variant>' -> one line of key metrics for the 3rd launch
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpc__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum -s 2 -c 1 --clock-control none --csv python tools/one_launch.py "$1" 2>/dev/null | python -c "
import csv,sys,json
rows=[r for r in csv.reader(sys.stdin) if len(r)>14 and r[0]!='ID']
print(json.dumps({'variant': sys.argv[1], **{r[12]: r[14] for r in rows}}))" "$1"
