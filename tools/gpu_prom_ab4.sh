#!/bin/bash
# per-operand L2 promotion rule vs the shipped 256B maps, odd and aligned leading dimensions
L=old=abl/lib_base256.so,new=paper_2108_13191_b200/libgemm_f16.so
for s in "8192 1000 1000" "4100 4096 4104" "4104 4104 4104" "8192 1024 1000" "2000 2000 2000" "3000 3000 3000" "8192 8192 8192"; do
  set -- $s
  M=$1 N=$2 K=$3 LIBS=$L ROUNDS=7 timeout 300 python tools/ab_libs.py
done
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_gemm_gpu_fuzz.py -x -q 2>&1 | tail -2
