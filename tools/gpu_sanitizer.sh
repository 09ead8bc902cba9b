for tool in memcheck racecheck synccheck initcheck; do
  for v in '{"M":512,"N":512,"K":512,"mode":"f32"}' '{"M":300,"N":264,"K":136,"mode":"f16"}' '{"M":300,"N":270,"K":200,"mode":"f32","config":"solo_128x64","pad":6}' '{"M":333,"N":261,"K":190,"mode":"f16","pad":11}' '{"M":256,"N":512,"K":2300,"mode":"f32","gather_peers":2}'; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/one_launch.py "$v" > gpurun_out/san_$tool.log 2>&1; rc=$?
    echo "$tool $v rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' gpurun_out/san_$tool.log | head -2 | tr '\n' ' ')"
  done
done
