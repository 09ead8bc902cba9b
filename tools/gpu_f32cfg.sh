#!/bin/bash
for sh in "16384 4096 1024" "4096 4096 1024" "32768 1024 1024" "8192 8192 2048" "12345 4096 1024" "8192 1000 1000"; do set -- $sh
VARIANTS='[{"mode":"f32","config":"pair_256x256_s5"},{"mode":"f32","config":"pair_256x256_k128"},{"mode":"f32","config":"pair_256x256"},{"mode":"f32","config":"pair_256x256_s4"}]' M=$1 N=$2 K=$3 ROUNDS=4 SECS=0.2 timeout 300 python tools/ab_power.py
done
