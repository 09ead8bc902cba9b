timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gputest.log | tail -15
timeout 900 python tools/ablation.py > gpurun_out/ablation_r01.jsonl 2> gpurun_out/ablation.err; echo "ablation rc=$?"; tail -2 gpurun_out/ablation.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
