python -m pytest tests/test_gemm_gpu.py -q -m gpu -x 2>&1 | tail -2
for sh in 8192x4096x1024 8192x8192x8192; do for c in 1 6 7; do python tools/trace_tiles.py $sh f32 "{\"config\": $c}" | tail -3; done; done
VARIANTS='[{"mode":"f32","config":1},{"mode":"f32","config":6},{"mode":"f32","config":7},{"mode":"f16","config":1},{"mode":"f16","config":6},{"mode":"f16","config":7}]' ROUNDS=5 python tools/ab.py
M=8192 N=4096 K=1024 VARIANTS='[{"mode":"f32","config":1},{"mode":"f32","config":6},{"mode":"f32","config":7},{"mode":"f16","config":1},{"mode":"f16","config":6},{"mode":"f16","config":7}]' ROUNDS=5 python tools/ab.py
