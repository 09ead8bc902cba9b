#!/bin/bash
for v in '{"M":300,"N":528,"K":777,"mode":"f16","config":"splitk_128x128_s4","pad":8}' '{"M":200,"N":300,"K":64,"mode":"f16","config":"splitk_128x128_s4"}' '{"M":300,"N":530,"K":1777,"mode":"f32","config":"splitk_128x128_s4","pad":8}'; do
  for tool in memcheck racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/one_launch.py "$v" > gpurun_out/san_$tool.log 2>&1; rc=$?
    echo "$tool $v rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | tr '\n' ' ')"
  done
done > gpurun_out/san6.txt
bash tools/gpu_final2.sh
cat gpurun_out/san6.txt
