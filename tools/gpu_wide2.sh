#!/bin/bash
# Wide-tile (256x512) F16 kernel vs the shipped pair_256x256_k128: per-tile traces, then power-regime A/B.
for c in pair_256x256_k128 pair_256x512; do
  timeout 120 python tools/trace_tiles.py 8192x8192x8192 f16 "{\"config\":\"$c\"}" 2>&1 | head -14
done > gpurun_out/wide_trace.txt
cat gpurun_out/wide_trace.txt
VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x512"}]' ROUNDS=8 SECS=0.3 timeout 600 python tools/ab_power.py 2>&1 | tee gpurun_out/wide_power.jsonl
VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x512"}]' ROUNDS=8 SECS=0.05 timeout 600 python tools/ab_power.py 2>&1 | tee -a gpurun_out/wide_power.jsonl
