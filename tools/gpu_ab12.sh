python -m pytest tests/test_gemm_gpu.py -q -m gpu -x -k "configs_ragged or phase_wrap or promotion_chunk" 2>&1 | tail -1
for c in 1 8; do python tools/trace_tiles.py 8192x8192x8192 f32 "{\"config\": $c}" 2>&1 | sed -n 5,7p | sed 's/.*| \([0-9]* cyc\)/\1/'; done
VARIANTS='[{"mode":"f32","config":1},{"mode":"f32","config":8},{"mode":"f16","config":1},{"mode":"f16","config":8}]' ROUNDS=6 python tools/ab.py
for v in '{"mode":"f32","config":1}' '{"mode":"f32","config":8}'; do bash tools/ncu_metrics.sh "$v"; done
