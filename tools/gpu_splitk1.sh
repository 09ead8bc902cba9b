#!/bin/bash
# Split-K cluster kernels: parity, then CUDA-graph GPU time per GEMM vs the existing small-shape configs.
timeout 900 python -m pytest tests/test_gemm_gpu_splitk.py -q -m gpu -x 2>&1 | tail -15
SHAPES=256x256x256,512x512x512,1024x1024x1024,1536x1536x1536,1024x1024x4096,2048x2048x512,4096x1024x1024 CFGS=1,5,6,10,11,12 timeout 600 python tools/graph_bench.py
