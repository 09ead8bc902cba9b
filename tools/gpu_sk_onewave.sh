#!/bin/bash
# stream-K below one wave (tiles split up to three ways): parity, then GPU time off/on
timeout 900 python -m pytest tests/test_gemm_gpu_streamk.py -x -q 2>&1 | tail -3
for o in '{"stream_k": -1}' '{"stream_k": 1}'; do
  echo "== $o"
  SHAPES=2048x2048x8192,1792x1792x8192,2048x2048x4096,1792x1792x4096,1792x1792x1792,2048x2048x2048,1536x2048x8192 \
  CFGS=7,8 OPTS="$o" timeout 600 python tools/graph_bench.py 2>&1
done
