#!/bin/bash
for sh in "32768 1024 1024" "8192 4096 1024" "12345 4096 1024" "4096 1024 1024" "32768 1024 4096" "8192 4096 4096"; do set -- $sh
VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x256_s5"},{"mode":"f16","config":"pair_256x256"},{"mode":"f16","config":"pair_256x512"}]' M=$1 N=$2 K=$3 ROUNDS=4 SECS=0.2 timeout 300 python tools/ab_power.py
done
