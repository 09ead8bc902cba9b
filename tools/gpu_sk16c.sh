#!/bin/bash
# F16: stream-K pair tile vs the 256x512 wide tile, interleaved rounds (ab_power), per shape
for s in "2304 2304 4096" "2560 2560 8192" "3840 3840 3840" "4608 4608 4608" "5120 5120 5120" "2304 2304 2304"; do
  set -- $s
  M=$1 N=$2 K=$3 ROUNDS=6 SECS=0.3 VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x512"},{"mode":"f16","config":"pair_256x256_k128","stream_k":-1}]' \
    timeout 300 python tools/ab_power.py
done
