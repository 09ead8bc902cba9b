#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -m gpu -x -k "c_reduce or ablation" 2>&1 | tail -3
VARIANTS='[{"mode":"f32"},{"mode":"f32","c_reduce":1}]' ROUNDS=6 SECS=0.3 timeout 900 python tools/ab_power.py
for sh in "16384 4096 1024" "8192 4096 1024" "4096 4096 1024" "8192 8192 2048" "32768 1024 1024" "16384 16384 16384"; do set -- $sh
VARIANTS='[{"mode":"f32"},{"mode":"f32","c_reduce":1}]' M=$1 N=$2 K=$3 ROUNDS=6 SECS=0.25 timeout 300 python tools/ab_power.py
done
VARIANTS='[{"mode":"f32"},{"mode":"f32","c_reduce":1}]' ROUNDS=10 REPS=6 timeout 600 python tools/ab.py
python tools/trace_tiles.py 16384x4096x1024 f32 '{"c_reduce":1}' 2>&1 | sed -n 3,9p
