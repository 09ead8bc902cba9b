#!/bin/bash
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_gemm_gpu_wide.py -q -m gpu -x -k "ablation or determin" 2>&1 | tail -2
VARIANTS='[{"mode":"f32"},{"mode":"f32","k_serpentine":2},{"mode":"f16"},{"mode":"f16","k_serpentine":2}]' ROUNDS=8 SECS=0.3 timeout 900 python tools/ab_power.py
VARIANTS='[{"mode":"f32"},{"mode":"f32","k_serpentine":2},{"mode":"f16"},{"mode":"f16","k_serpentine":2}]' M=16384 ROUNDS=4 SECS=0.4 timeout 900 python tools/ab_power.py
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -s 4 -c 4 python tools/one_launch.py '{"mode":"f32"}' 2>/dev/null | grep -E "dram__bytes|duration" 
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -s 4 -c 4 python tools/one_launch.py '{"mode":"f32","k_serpentine":2}' 2>/dev/null | grep -E "dram__bytes|duration"
