timeout 600 ncu --set full --clock-control none -s 2 -c 1 -o gpurun_out/prof_cublas -f python tools/prof_cublas.py > gpurun_out/prof_cublas.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/prof_cublas.log
