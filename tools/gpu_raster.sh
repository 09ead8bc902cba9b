MODE=f32 python tools/sweep_raster.py
MODE=f16 python tools/sweep_raster.py
for gm in 2 8 32; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,gpc__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none --csv python - <<PY 2>/dev/null | grep -E "dram__bytes_read|gpc__cycles|time_duration|hit_rate" | tail -4 | sed "s/^/gm=$gm /"
import os, sys; sys.path.insert(0, "."); import torch, synth, paper_2108_13191_b200 as g
n=8192; A=torch.from_numpy(synth.uniform_f16(0,0,n,n)).cuda(); B=torch.from_numpy(synth.uniform_f16(0,1,n,n)).cuda(); C=torch.from_numpy(synth.uniform_f32(0,2,n,n)).cuda()
g.gemm_f16(A,B,C,group_m=$gm); torch.cuda.synchronize()
PY
done
