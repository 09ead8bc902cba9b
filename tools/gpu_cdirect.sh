#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -m gpu -x -k "ablation" 2>&1 | tail -2
VARIANTS='[{"mode":"f32"},{"mode":"f32","c_store":1},{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x256_k128","c_store":1}]' ROUNDS=6 SECS=0.3 timeout 900 python tools/ab_power.py
for sh in "16384 4096 1024" "8192 8192 2048"; do set -- $sh
VARIANTS='[{"mode":"f32"},{"mode":"f32","c_store":1}]' M=$1 N=$2 K=$3 ROUNDS=6 SECS=0.25 timeout 300 python tools/ab_power.py
done
python tools/trace_tiles.py 8192x8192x8192 f32 '{"c_store":1}' 2>&1 | sed -n 3,10p
