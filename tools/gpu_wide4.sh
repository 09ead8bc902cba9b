#!/bin/bash
# Split-half wide kernel: parity, traces, power-regime A/B vs k128.
timeout 300 python -m pytest tests/test_gemm_gpu_wide.py -q -m gpu -x 2>&1 | tail -3
timeout 120 python tools/trace_tiles.py 8192x8192x8192 f16 '{"config":"pair_256x512"}' 2>&1 | sed -n 3,10p
timeout 120 python tools/trace_tiles.py 16384x4096x4096 f16 '{"config":"pair_256x512"}' 2>&1 | sed -n 3,8p
VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x512"}]' ROUNDS=8 SECS=0.3 timeout 600 python tools/ab_power.py
VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x512"}]' M=16384 N=4096 K=4096 ROUNDS=6 SECS=0.3 timeout 600 python tools/ab_power.py
VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x512"}]' M=4096 ROUNDS=6 SECS=0.3 timeout 600 python tools/ab_power.py
VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x512"}]' ROUNDS=10 REPS=6 timeout 600 python tools/ab.py
