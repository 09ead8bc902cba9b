#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; cat gpurun_out/bench2.json
