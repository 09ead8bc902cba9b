timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gputest.log | tail -15
timeout 600 python bench.py --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
VARIANTS='[{"mode":"f32"},{"mode":"f32","promote_k":-1},{"mode":"f16"},{"mode":"f16","promote_k":-1}]' ROUNDS=4 python tools/ab.py
for v in '{"mode":"f32"}' '{"mode":"f32","promote_k":-1}'; do bash tools/ncu_metrics.sh "$v"; done
