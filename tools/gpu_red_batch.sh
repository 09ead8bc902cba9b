#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu_splitk.py -q -m gpu -x 2>&1 | tail -2
python tools/trace_splitk.py 1024x1024x1024:f16:splitk_128x128_s2 512x512x2048:f16:splitk_128x128_s4
SHAPES=1024x1024x1024,1024x1024x2048,512x512x2048,256x1024x16384,1024x1024x4096,768x768x2048 CFGS=0,5,12,15 timeout 600 python tools/graph_bench.py
