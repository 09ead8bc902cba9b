#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -m gpu -x -k "ablation or determin or ragged or closed or brute or small_integers or c_reduce or pdl" 2>&1 | tail -3
for sh in "8192 8192 8192" "4096 4096 4096" "2304 2304 2304" "2560 2560 2560" "3840 3840 3840" "12288 12288 12288"; do set -- $sh
LIBS=prev=tools/libgemm_prev.so,sk=tools/libgemm_sk.so MODES=f32 M=$1 N=$2 K=$3 ROUNDS=8 REPS=$((2000000000000 / ($1*$2*$3) + 3)) timeout 300 python tools/ab_libs.py
done
