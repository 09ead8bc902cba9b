#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu_splitk.py -q -m gpu -x 2>&1 | tail -4
python tools/trace_splitk.py 1024x1024x1024:f16:splitk_128x256_s4 1024x1024x1024:f32:splitk_128x256_s4 256x256x256:f16:splitk_128x256_s2 1024x1024x4096:f16:splitk_128x256_s4 1024x1024x1024:f32:splitk_128x128_s4
SHAPES=256x256x256,512x512x512,1024x1024x1024,1024x1024x4096,512x512x2048,1024x1024x2048,2048x1024x1024 CFGS=5,6,10,11,12 timeout 600 python tools/graph_bench.py
