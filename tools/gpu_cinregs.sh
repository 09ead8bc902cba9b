#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -m gpu -x -k "cin_regs or ablation or ragged or closed or brute or small_integers" 2>&1 | tail -2
for sh in "16384 4096 1024" "8192 4096 1024" "32768 1024 1024" "4096 4096 1024" "8192 8192 2048" "12345 4096 1024"; do set -- $sh
VARIANTS='[{"mode":"f32"},{"mode":"f32","cin_regs":-1}]' M=$1 N=$2 K=$3 ROUNDS=6 SECS=0.25 timeout 300 python tools/ab_power.py
done
python tools/trace_tiles.py 16384x4096x1024 f32 2>&1 | sed -n 3,9p
python tools/trace_tiles.py 16384x4096x1024 f32 '{"cin_regs":-1}' 2>&1 | sed -n 3,9p
