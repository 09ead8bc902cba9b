#!/bin/bash
# A/B of the L2 promotion per operand (A only / B only at 128B) on odd-leading-dimension shapes
L=base=paper_2108_13191_b200/libgemm_f16.so,p128=abl/lib_prom128.so,pA=abl/lib_pA128.so,pB=abl/lib_pB128.so
for s in "8192 1000 1000" "4100 4096 4104" "8192 1000 4000" "8192 1024 1000" "8192 4000 4000" "4104 4104 4104"; do
  set -- $s
  M=$1 N=$2 K=$3 LIBS=$L ROUNDS=7 timeout 300 python tools/ab_libs.py
done
