#!/bin/bash
# A/B of the L2 promotion on more odd-leading-dimension shapes (short and mid K)
L=base=paper_2108_13191_b200/libgemm_f16.so,p128=abl/lib_prom128.so
for s in "16384 1000 1000" "8000 4000 1000" "4000 1000 1000" "8192 1000 512" "8192 1000 2000" "8192 3000 1000" "8192 1000 4000" "8192 4000 4000"; do
  set -- $s
  M=$1 N=$2 K=$3 LIBS=$L ROUNDS=7 timeout 300 python tools/ab_libs.py
done
