#!/bin/bash
# ncu full capture of the 256x512 F16 kernel at 8192^3 + the bench launch list.
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wide -s 2 -c 1 -o gpurun_out/r01_wide_f16_8192 -f python tools/prof_one.py --modes f16 > /dev/null 2>&1; echo "rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_wide_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1; echo "rc=$?"
