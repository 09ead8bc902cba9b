#!/bin/bash
# DIAGNOSTIC: F32 K=1024 memory behaviour + knob A/B
for v in '{"M":16384,"N":4096,"K":1024,"config":"pair_256x256_s5"}' \
         '{"M":16384,"N":4096,"K":1024,"config":"pair_256x256_s5","beta":0}' \
         '{"M":16384,"N":4096,"K":1024,"config":"pair_256x256_s5","l2_hints":0}' \
         '{"M":16384,"N":4096,"K":1024,"mode":"f16","config":"pair_256x256_k128"}'; do
  bash tools/ncu_metrics.sh "$v"
done
M=16384 N=4096 K=1024 ROUNDS=7 REPS=20 VARIANTS='[{"mode":"f32","config":"pair_256x256_s5"},{"mode":"f32","config":"pair_256x256_k128"},{"mode":"f32","config":"pair_256x256_s5","l2_hints":0},{"mode":"f32","config":"pair_256x256_s5","c_row_prefetch":1},{"mode":"f32","config":"pair_256x256_s5","group_m":4},{"mode":"f32","config":"pair_256x256_s5","group_m":16},{"mode":"f32","config":"pair_256x256_s5","epi_pace":1},{"mode":"f32","config":"pair_256x256_s4"},{"mode":"f32","config":"pair_256x256"},{"mode":"f32","config":"pair_256x128"},{"mode":"f32","config":"pair_256x256_s5","max_clusters":64},{"mode":"f32","config":"pair_256x256_s5","beta":0}]' python tools/ab.py
