#!/bin/bash
# stream-K run boundaries snapped to tile edges (k_blocks / 8, at least one full wave): parity, then
# snapped build vs stream-K off vs the previous build's numbers (profiles/r01/stream_k/snap_experiment.txt)
timeout 900 python -m pytest tests/test_gemm_gpu_streamk.py tests/test_gemm_gpu_fuzz.py -x -q 2>&1 | tail -1
for o in '{}' '{"stream_k": -1}'; do
  echo "== $o"
  SHAPES=2304x2304x2304,3840x3840x3840,3328x3328x3328,2304x2304x8192,1792x1792x8192 CFGS=0 OPTS="$o" timeout 600 python tools/graph_bench.py 2>&1
done
