#!/bin/bash
# wide-kernel tail ring: parity, then old/new build A/B on wide-picked F16 shapes
timeout 900 python -m pytest tests/test_gemm_gpu_wide.py -x -q 2>&1 | tail -2
L=old=abl/lib_base256.so,new=paper_2108_13191_b200/libgemm_f16.so
for s in "2816 2816 2816" "4096 4096 4096" "3072 3072 2048" "8192 1024 1024" "16384 1024 1024"; do
  set -- $s
  M=$1 N=$2 K=$3 MODES=f16 LIBS=$L ROUNDS=7 timeout 300 python tools/ab_libs.py
done
MODES=f16 SHAPES=2816x2816x2816,4096x4096x4096,8192x1024x1024 CFGS=9 OPTS='{"tail_ring": -1}' timeout 300 python tools/graph_bench.py
MODES=f16 SHAPES=2816x2816x2816,4096x4096x4096,8192x1024x1024 CFGS=9 timeout 300 python tools/graph_bench.py
