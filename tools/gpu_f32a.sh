#!/bin/bash
# F32 mode: per-tile trace and power-regime A/B of scheduling knobs.
timeout 120 python tools/trace_tiles.py 8192x8192x8192 f32 2>&1 | sed -n 3,12p
VARIANTS='[{"mode":"f32"},{"mode":"f32","promote_k":4096},{"mode":"f32","group_m":16},{"mode":"f32","l2_hints":-1},{"mode":"f16","config":"pair_256x256_k128"}]' ROUNDS=6 SECS=0.3 timeout 600 python tools/ab_power.py
