#!/bin/bash
# A/B: c_row_prefetch=2 (producer prefetches next tile's C_in) on K=1024 shapes and 8192^3
V='[{"mode":"f32","config":"pair_256x256_s5"},{"mode":"f32","config":"pair_256x256_s5","c_row_prefetch":2},{"mode":"f32","config":"pair_256x256_k128","c_row_prefetch":2},{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x256_k128","c_row_prefetch":2}]'
M=16384 N=4096 K=1024 ROUNDS=7 REPS=20 VARIANTS="$V" python tools/ab.py
M=8192 N=4096 K=1024 ROUNDS=7 REPS=20 VARIANTS="$V" python tools/ab.py
M=4096 N=4096 K=1024 ROUNDS=7 REPS=20 VARIANTS="$V" python tools/ab.py
V='[{"mode":"f32"},{"mode":"f32","c_row_prefetch":2},{"mode":"f16"},{"mode":"f16","c_row_prefetch":2}]'
M=8192 ROUNDS=7 REPS=10 VARIANTS="$V" python tools/ab.py
M=4096 ROUNDS=7 REPS=20 VARIANTS="$V" python tools/ab.py
