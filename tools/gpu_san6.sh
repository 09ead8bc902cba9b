#!/bin/bash
# compute-sanitizer over the stream-K schedule (token hand-over between clusters) and the
# tail-ring staging of the last tile
for tool in memcheck racecheck synccheck initcheck; do
  for v in '{"M":1300,"N":2100,"K":640,"mode":"f32","config":"pair_256x256","max_clusters":5,"stream_k":1}' \
           '{"M":1000,"N":1032,"K":4200,"mode":"f32","config":"pair_256x256_k128","max_clusters":3,"stream_k":1}' \
           '{"M":770,"N":776,"K":3000,"mode":"f32","config":"pair_256x256_s4","max_clusters":3,"stream_k":1}' \
           '{"M":700,"N":900,"K":500,"mode":"f16","config":"pair_256x256","beta":0}'; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/one_launch.py "$v" > gpurun_out/san_$tool.log 2>&1; rc=$?
    echo "$tool $v rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' gpurun_out/san_$tool.log | head -2 | tr '\n' ' ')"
  done
done
