#!/bin/bash
# F16 stream-K: parity, then GPU time off/on for the pair configs vs the wide tile
timeout 900 python -m pytest tests/test_gemm_gpu_streamk.py -x -q 2>&1 | tail -3
for o in '{"stream_k": -1}' '{"stream_k": 1}'; do
  echo "== $o"
  MODES=f16 SHAPES=2304x2304x2304,2304x2304x4096,2304x2304x8192,2560x2560x8192,3840x3840x3840,4096x4096x4096,4608x4608x4608,2816x2816x8192 \
  CFGS=1,8,9 OPTS="$o" timeout 600 python tools/graph_bench.py 2>&1
done
