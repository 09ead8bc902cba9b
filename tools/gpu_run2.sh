set -x
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -m gpu > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_one.py --warmup 1 > /dev/null 2>&1; echo "ncu rc=$?"
cat gpurun_out/launches.csv | tail -30
