#!/bin/bash
# stream-K parity + the full GPU suite subset touching the pair kernels, and an A/B of the default bench shape
timeout 900 python -m pytest tests/test_gemm_gpu_streamk.py tests/test_gemm_gpu.py tests/test_gemm_gpu_epilogue.py tests/test_gemm_gpu_fuzz.py -x -q 2>&1 | tail -4
SHAPES=2304x2304x4096,3840x3840x3840,2048x2048x2048,1792x1792x1792 CFGS=0 timeout 600 python tools/graph_bench.py 2>&1 | grep '"f32"'
timeout 600 python bench.py 2>&1 | tail -1
