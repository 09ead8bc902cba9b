#!/bin/bash
# stream-K on/off over square and long-K shapes (auto config, F32, CUDA-graph replay)
S=""
for n in 2304 2560 2816 3072 3328 3584 3840 4096 4352 4608 4864 5120 5376 5632 5888 6144; do S="$S,${n}x${n}x${n}"; done
for n in 2304 2560 2816 3072 3584 4096; do S="$S,${n}x${n}x8192"; done
S="$S,2304x2304x4096,3840x3840x1024,4608x4608x2048,8192x8192x8192"
S=${S#,}
for o in '{"stream_k": -1}' '{"stream_k": 1}'; do
  echo "== $o"
  SHAPES=$S CFGS=0 OPTS="$o" timeout 900 python tools/graph_bench.py 2>&1 | grep '"f32"'
done
