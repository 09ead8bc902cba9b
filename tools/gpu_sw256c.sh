HI=6144 timeout 1700 python tools/sweep256.py > gpurun_out/sweep256_c.jsonl 2> gpurun_out/sweep256_c.err; echo rc=$?
