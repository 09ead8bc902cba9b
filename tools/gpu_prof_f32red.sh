#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f16_sm100_kernel -s 2 -c 1 -o gpurun_out/r01_f32_reduce_8192 -f python tools/prof_one.py --modes f32 > /dev/null 2>&1; echo "rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:gemm_f16_sm100_kernel -s 2 -c 1 -o gpurun_out/r01_f32_reduce_16384x4096x1024 -f python tools/prof_one.py --modes f32 --m 16384 --n 4096 --k 1024 > /dev/null 2>&1; echo "rc=$?"
