python -m pytest tests/test_gemm_gpu.py -q -m gpu -x -k "ragged or brute or ablation" 2>&1 | tail -1
for sh in "8192 4096 1024" "16384 4096 1024" "32768 1024 1024" "8192 8192 8192"; do set -- $sh; M=$1 N=$2 K=$3 VARIANTS='[{"mode":"f32"},{"mode":"f32","c_row_prefetch":1},{"mode":"f16"},{"mode":"f16","c_row_prefetch":1}]' ROUNDS=8 REPS=$((1000000000000 / ($1*$2*$3) + 3)) python tools/ab.py; done
python tools/trace_tiles.py 8192x4096x1024 f32 '{"c_row_prefetch":1}' 2>&1 | sed -n 4,8p
