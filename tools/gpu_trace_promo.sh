#!/bin/bash
for kw in '{}' '{"promote_k":-1}' '{"promote_k":4096}' '{"debug_flags":3}' '{"debug_flags":3,"promote_k":-1}'; do
python tools/trace_tiles.py 8192x8192x8192 f32 "$kw" 2>&1 | sed -n 3,12p | awk '{print $0}' | grep -o "^.*cyc per k-block\|^8192.*" | tail -9
done
python tools/trace_tiles.py 8192x8192x8192 f16 '{"config":"pair_256x256_k128"}' 2>&1 | sed -n 3,12p
python tools/trace_tiles.py 8192x8192x8192 f16 '{"config":"pair_256x256_k128","promote_k":-1}' 2>&1 | sed -n 3,12p
