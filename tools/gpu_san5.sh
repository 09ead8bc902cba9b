#!/bin/bash
for v in '{"M":300,"N":528,"K":777,"mode":"f32","config":"splitk_128x256_s4","pad":8}' '{"M":260,"N":512,"K":2100,"mode":"f32","config":"splitk_128x256_s2"}' '{"M":200,"N":300,"K":64,"mode":"f32","config":"splitk_128x128_s4"}' '{"M":777,"N":1000,"K":1000,"mode":"f32","config":"pair_256x256_k128"}'; do
  for tool in memcheck racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/one_launch.py "$v" > gpurun_out/san_$tool.log 2>&1; rc=$?
    echo "$tool $v rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | tr '\n' ' ') $(grep -oE 'in [A-Za-z_.]+:[0-9]+' gpurun_out/san_$tool.log | sort -u | head -3 | tr '\n' ' ')"
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
