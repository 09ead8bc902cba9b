#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu_splitk.py tests/test_gemm_gpu.py -q -m gpu -x -k "splitk or pdl_mixed" 2>&1 | tail -3
python tools/trace_splitk.py 512x512x2048:f16:splitk_128x128_s4 512x512x8192:f16:splitk_128x128_s4
SHAPES=256x1024x16384,512x512x8192,256x256x4096,128x4096x4096,512x512x2048 CFGS=0,12 timeout 600 python tools/graph_bench.py
