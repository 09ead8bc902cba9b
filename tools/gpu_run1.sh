set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 120 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -20 gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -m gpu > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/gputest.log
