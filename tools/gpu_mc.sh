#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -m gpu -x -k "multicast or ragged_multi or phase_wrap or small_integers" 2>&1 | tail -3
SHAPES=256x256x256,512x512x512,1024x1024x1024,1024x1024x2048,2048x1024x1024,512x2048x1024 CFGS=0,5,4,13,14 timeout 600 python tools/graph_bench.py
