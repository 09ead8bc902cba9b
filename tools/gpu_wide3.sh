#!/bin/bash
# Wide kernel with the lean drain: traces, drain variant A/B (library builds), power-regime A/B vs k128.
timeout 300 python -m pytest tests/test_gemm_gpu_wide.py -q -m gpu -x 2>&1 | tail -3
for c in pair_256x512; do
  timeout 120 python tools/trace_tiles.py 8192x8192x8192 f16 "{\"config\":\"$c\"}" 2>&1 | sed -n 3,10p
done
LIBS=db=tools/libgemm_db.so,single=tools/libgemm_single.so MODES=f16 ROUNDS=10 REPS=10 timeout 300 python tools/ab_libs.py
VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x512"}]' ROUNDS=8 SECS=0.3 timeout 600 python tools/ab_power.py
VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x512"}]' M=16384 N=4096 K=4096 ROUNDS=6 SECS=0.3 timeout 600 python tools/ab_power.py
VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x512"}]' M=4096 ROUNDS=6 SECS=0.3 timeout 600 python tools/ab_power.py
