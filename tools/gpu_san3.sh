#!/bin/bash
# compute-sanitizer over the wide (256x512) and split-K kernels on small ragged shapes.
for v in '{"M":600,"N":1100,"K":700,"mode":"f16","config":"pair_256x512","pad":8}' \
         '{"M":520,"N":1030,"K":300,"mode":"f16","config":"pair_256x512","max_clusters":1}' \
         '{"M":300,"N":530,"K":777,"mode":"f32","config":"splitk_128x256_s4","pad":8}' \
         '{"M":300,"N":530,"K":777,"mode":"f16","config":"splitk_128x128_s4","pad":8}' \
         '{"M":260,"N":515,"K":2100,"mode":"f32","config":"splitk_128x256_s2"}' \
         '{"M":200,"N":300,"K":64,"mode":"f32","config":"splitk_128x256_s4"}'; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/one_launch.py "$v" > gpurun_out/san_$tool.log 2>&1; rc=$?
    echo "$tool $v rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | tr '\n' ' ') $(grep -oE '(Read|Write) access at [^ ]+ [^ ]+ in [A-Za-z_.]+:[0-9]+' gpurun_out/san_$tool.log | sort -u | head -3 | tr '\n' ' ')"
  done
done
