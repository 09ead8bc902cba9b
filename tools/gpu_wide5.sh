#!/bin/bash
# F16 config choice: pair_256x256 family vs pair_256x512 over BASELINE shapes (power-regime A/B).
for sh in "2048 2048 2048" "4096 4096 4096" "6144 6144 6144" "8192 8192 8192" "12288 12288 12288" "16384 16384 16384" \
          "4096 1024 1024" "4096 4096 1024" "8192 1024 4096" "16384 4096 4096" "32768 1024 4096" "12345 4096 1024" \
          "8192 8192 2048" "8192 8192 1024" "8192 1000 1000" "4100 4096 4104"; do
  set -- $sh
  VARIANTS='[{"mode":"f16"},{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x256_s5"},{"mode":"f16","config":"pair_256x512"}]' M=$1 N=$2 K=$3 ROUNDS=4 SECS=0.15 timeout 300 python tools/ab_power.py
done
