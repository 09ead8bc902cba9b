#!/bin/bash
# ncu full capture of the stream-K pair kernels (F32 and F16) at 2304^2 x 8192 -- the shape
# where stream-K gains most -- and of the data-parallel kernel at the same shape for contrast
for v in '{"M":2304,"N":2304,"K":8192,"mode":"f32","config":"pair_256x256_k128","stream_k":1}' \
         '{"M":2304,"N":2304,"K":8192,"mode":"f32","config":"pair_256x256_k128","stream_k":-1}' \
         '{"M":2304,"N":2304,"K":8192,"mode":"f16","config":"pair_256x256_k128","stream_k":1}'; do
  tag=$(echo "$v" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['mode'] + ('_sk' if d['stream_k']>0 else '_dp'))")
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f16_sm100_kernel -s 2 -c 1 -o gpurun_out/r01_sk_2304x8192_$tag -f python tools/one_launch.py "$v" > /dev/null 2>&1; echo "$tag rc=$?"
done
