#!/bin/bash
# EXPERIMENT: snapping stream-K run boundaries to tile edges (GEMM_SK_SNAP_DIV = k_blocks / snap)
timeout 600 python -m pytest tests/test_gemm_gpu_streamk.py -x -q 2>&1 | tail -1
for div in 0 8 4; do
  echo "== div $div"
  GEMM_SK_SNAP_DIV=$div GEMM_SK_SNAP=1 SHAPES=2304x2304x2304,3840x3840x3840,4608x4608x4608,2304x2304x8192,3328x3328x3328,1792x1792x8192 \
    CFGS=0 timeout 600 python tools/graph_bench.py 2>&1
done
GEMM_SK_SNAP_DIV=4 timeout 600 python -m pytest tests/test_gemm_gpu_streamk.py -x -q 2>&1 | tail -1
