#!/bin/bash
# F16 stream-K pick rule: parity suite, then auto vs the previous picks (wide / k128 DP)
timeout 1500 python -m pytest tests/test_gemm_gpu_streamk.py tests/test_gemm_gpu_wide.py tests/test_gemm_gpu_fuzz.py tests/test_gemm_gpu.py -x -q 2>&1 | tail -3
MODES=f16 SHAPES=2304x2304x2304,2304x2304x4096,2560x2560x8192,3840x3840x3840,4096x4096x4096,4608x4608x4608,5120x5120x5120,2816x2816x2816 \
  CFGS=0,8,9 timeout 600 python tools/graph_bench.py 2>&1
