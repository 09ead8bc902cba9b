#!/bin/bash
# one-wave stream-K auto rule: auto (default) vs auto with stream-K off
timeout 900 python -m pytest tests/test_gemm_gpu_streamk.py tests/test_gemm_gpu_fuzz.py tests/test_gemm_gpu.py -x -q 2>&1 | tail -2
for o in '{"stream_k": -1}' '{}'; do
  echo "== $o"
  SHAPES=2048x2048x8192,1792x1792x8192,1792x1792x4096,1536x2048x8192,1792x1792x1792,2048x2048x4096,1536x1536x16384 \
  CFGS=0 OPTS="$o" timeout 600 python tools/graph_bench.py 2>&1
done
