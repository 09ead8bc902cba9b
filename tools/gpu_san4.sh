timeout 600 compute-sanitizer --tool racecheck --print-level info python tools/one_launch.py '{"M":600,"N":1100,"K":700,"mode":"f16","config":"pair_256x512","pad":8}' > gpurun_out/san_rc_wide.log 2>&1
grep -v "^=========     Host Frame\|^=========         in \|^=========     Saved host" gpurun_out/san_rc_wide.log | head -60
