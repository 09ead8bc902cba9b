#!/bin/bash
# compute-sanitizer over stream-K below one wave (tiles split three ways; middle parts wait and post)
for tool in memcheck racecheck synccheck; do
  for v in '{"M":700,"N":704,"K":2000,"mode":"f32","config":"pair_256x256","max_clusters":12,"stream_k":1}' \
           '{"M":600,"N":1000,"K":1500,"mode":"f16","config":"pair_256x256_k128","max_clusters":10,"stream_k":1}'; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/one_launch.py "$v" > gpurun_out/san_$tool.log 2>&1; rc=$?
    echo "$tool $v rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | head -1)"
  done
done
