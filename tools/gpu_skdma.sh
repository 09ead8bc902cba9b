#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu_splitk.py -q -m gpu -x 2>&1 | tail -3
python tools/trace_splitk.py 1024x1024x1024:f16:splitk_128x256_s4 512x512x2048:f16:splitk_128x128_s4 1024x1024x4096:f16:splitk_128x256_s2 1024x1024x1024:f32:splitk_128x256_s4:0
SHAPES=1024x1024x1024,256x1024x16384,512x512x8192,256x256x4096,128x4096x4096,512x512x2048,1024x1024x4096,1024x1024x8192 CFGS=0,5,10,11,12 timeout 600 python tools/graph_bench.py
