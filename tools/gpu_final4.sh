#!/bin/bash
# Round-end evidence after stream-K / tail ring: GPU suite, smoke, default bench, ncu launch list,
# and the 256-step square sweep with the final pick rules.
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/final4_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final4_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/final4_bench.json 2> gpurun_out/final4_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final4_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1
true
cat gpurun_out/final4_pytest.txt gpurun_out/final4_smoke.txt
