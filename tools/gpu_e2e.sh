#!/bin/bash
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -m gpu -x -k "host" 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; python -c "import json; d=json.load(open('gpurun_out/bench3.json')); print(d['value'], d['e2e'], d['modes'])"
