#!/bin/bash
# stream-K: parity tests, then GPU time (CUDA-graph replay) with the schedule off / on
timeout 900 python -m pytest tests/test_gemm_gpu_streamk.py -x -q 2>&1 | tail -3
for o in '{"stream_k": -1}' '{"stream_k": 1}'; do
  echo "== $o"
  SHAPES=${SHAPES:-2304x2304x2304,2560x2560x2560,1792x1792x1792,4096x4096x4096,3840x3840x3840,4608x4608x4608,2304x2304x8192} \
  CFGS=${CFGS:-1,8} OPTS="$o" timeout 600 python tools/graph_bench.py 2>&1 | grep '"f32"'
done
