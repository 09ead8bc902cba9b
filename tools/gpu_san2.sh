for v in '{"M":1024,"N":1024,"K":512,"mode":"f32","config":"pair_256x256_k128"}' '{"M":1024,"N":1024,"K":512,"mode":"f16","config":"pair_256x256"}' '{"M":1024,"N":1024,"K":512,"mode":"f32","config":"solo_128x256"}' '{"M":1024,"N":1024,"K":2300,"mode":"f32","config":"pair_256x256_s5"}'; do
  timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/one_launch.py "$v" > gpurun_out/san_rc.log 2>&1; rc=$?
  echo "racecheck $v rc=$rc $(grep -E 'RACECHECK SUMMARY' gpurun_out/san_rc.log | tr '\n' ' ') $(grep -oE 'Read access at [^ ]+ [^ ]+ in [a-z_.]+:[0-9]+' gpurun_out/san_rc.log | sort -u | head -2 | tr '\n' ' ')"
  timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/one_launch.py "$v" > gpurun_out/san_mc.log 2>&1; echo "memcheck rc=$? $(grep 'ERROR SUMMARY' gpurun_out/san_mc.log)"
done
