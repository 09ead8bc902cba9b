#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu_splitk.py -q -m gpu -x 2>&1 | tail -2
SHAPES=1024x1024x16384,1024x1024x1024,768x768x2048 CFGS=0,5,11,15 timeout 600 python tools/graph_bench.py
