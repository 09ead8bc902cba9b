# full ncu capture of one 8192^3 launch per mode (after warm-up)
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f16 -s 2 -c 1 -o gpurun_out/prof_f32 -f python tools/prof_one.py --modes f32 --warmup 2 > gpurun_out/prof_f32.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/prof_f32.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f16 -s 2 -c 1 -o gpurun_out/prof_f16 -f python tools/prof_one.py --modes f16 --warmup 2 > gpurun_out/prof_f16.log 2>&1; echo "rc=$?"
ls -la gpurun_out/
