#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu_splitk.py -q -m gpu -x 2>&1 | tail -2
SHAPES=1024x1024x4096,1024x2048x4096,1024x1024x2048 CFGS=0,10,11 timeout 600 python tools/graph_bench.py
