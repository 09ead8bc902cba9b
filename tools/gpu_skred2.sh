#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu_splitk.py -q -m gpu -x 2>&1 | tail -2
SHAPES=256x1024x16384,512x512x8192,256x256x4096,1024x1024x8192 CFGS=0,5,12 timeout 600 python tools/graph_bench.py
