#!/bin/bash
# Round-end evidence, final build: GPU suite, smoke, default bench, ncu launch list of the bench,
# the 256-step square sweep to 6144 and the BASELINE configs sweep.
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/final6_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/final6_bench.json 2> gpurun_out/final6_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final6_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1
cat gpurun_out/final6_pytest.txt gpurun_out/final6_smoke.txt
