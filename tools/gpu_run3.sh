timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
