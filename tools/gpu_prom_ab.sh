#!/bin/bash
# A/B: TMA L2 promotion of the A/B operand maps (256B shipped / 128B / none), one process per shape
L=base=paper_2108_13191_b200/libgemm_f16.so,p128=abl/lib_prom128.so,pnone=abl/lib_promnone.so
for s in "8192 1000 1000" "8192 1024 1024" "4100 4096 4104" "2000 2000 2000"; do
  set -- $s
  M=$1 N=$2 K=$3 LIBS=$L ROUNDS=7 timeout 300 python tools/ab_libs.py
done
M=8192 LIBS=$L ROUNDS=5 REPS=10 timeout 300 python tools/ab_libs.py
