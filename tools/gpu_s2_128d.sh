#!/bin/bash
timeout 1200 python -m pytest tests/test_gemm_gpu_splitk.py tests/test_gemm_gpu.py -q -m gpu -x 2>&1 | tail -3
for v in '{"M":300,"N":528,"K":777,"mode":"f16","config":"splitk_128x128_s2","pad":8}' '{"M":300,"N":528,"K":777,"mode":"f32","config":"splitk_128x128_s2","pad":8}'; do
  for tool in racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/one_launch.py "$v" > gpurun_out/san_$tool.log 2>&1; rc=$?
    echo "$tool $v rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | tr '\n' ' ')"
  done
done
