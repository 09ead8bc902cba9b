timeout 2000 python tools/sweep.py > gpurun_out/sweep_baseline_b.jsonl 2> gpurun_out/sweep_baseline_b.err; echo rc=$?
