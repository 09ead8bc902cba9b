#!/bin/bash
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_gemm_gpu_wide.py -q -m gpu -x -k "ablation or determin" 2>&1 | tail -2
VARIANTS='[{"mode":"f32"},{"mode":"f32","raster":1},{"mode":"f32","raster":1,"group_m":4},{"mode":"f16"},{"mode":"f16","raster":1},{"mode":"f16","raster":1,"group_m":4}]' ROUNDS=6 SECS=0.3 timeout 900 python tools/ab_power.py
VARIANTS='[{"mode":"f32"},{"mode":"f32","raster":1},{"mode":"f16"},{"mode":"f16","raster":1}]' M=16384 ROUNDS=4 SECS=0.4 timeout 900 python tools/ab_power.py
