timeout 900 python -m pytest tests/test_gemm_gpu.py -q -m gpu -x 2>&1 | grep -E "FAILED|Error|error|assert" | head -20
