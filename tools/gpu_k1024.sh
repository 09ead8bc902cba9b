#!/bin/bash
# DIAGNOSTIC: why F32 mode at K=1024 sits at ~0.58 of roofline
set -x
S=16384x4096x1024
python tools/trace_tiles.py $S f32 '{"config":"pair_256x256_s5"}' 2>&1 | head -30
python tools/trace_tiles.py $S f32 '{"config":"pair_256x256_k128"}' 2>&1 | head -30
python tools/trace_tiles.py $S f16 '{"config":"pair_256x256_k128"}' 2>&1 | head -30
python tools/trace_tiles.py $S f32 '{"config":"pair_256x256_s5","beta":0}' 2>&1 | head -30
