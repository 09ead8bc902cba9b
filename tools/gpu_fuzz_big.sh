FUZZ_EXTRA=300 timeout 1500 python -m pytest tests/test_gemm_gpu_fuzz.py -q -m gpu -x 2>&1 | tail -4
