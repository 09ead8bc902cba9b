#!/bin/bash
# Round-end evidence, final build: GPU suite, smoke, default bench, ncu launch list of the bench,
# the 256-step square sweep to 6144 and the BASELINE configs sweep.
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/final5_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final5_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/final5_bench.json 2> gpurun_out/final5_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final5_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1
HI=6144 timeout 900 python tools/sweep256.py > gpurun_out/final5_sweep256.jsonl 2> gpurun_out/final5_sweep256.err
timeout 1400 python tools/sweep.py > gpurun_out/final5_sweep_baseline.jsonl 2> gpurun_out/final5_sweep_baseline.err
cat gpurun_out/final5_pytest.txt gpurun_out/final5_smoke.txt
