#!/bin/bash
# First GPU pass of the 256x512 F16 kernel: its parity tests, then A/B vs the shipped F16 config.
timeout 900 python -m pytest tests/test_gemm_gpu_wide.py -q -m gpu -x 2>&1 | tail -25 > gpurun_out/wide_tests.log
cat gpurun_out/wide_tests.log
for sh in "8192 8192 8192" "16384 16384 16384" "4096 4096 4096" "16384 4096 4096" "8192 8192 2048"; do set -- $sh
  M=$1 N=$2 K=$3 VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x512"},{"mode":"f16","config":"pair_256x512","ring_stages":3}]' ROUNDS=6 REPS=$((2000000000000 / ($1*$2*$3) + 3)) timeout 300 python tools/ab.py
done 2>&1 | tee gpurun_out/wide_ab.jsonl
