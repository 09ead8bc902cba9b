#!/bin/bash
# stream-K timeline at 3840^3 F32 (pair_256x256_k128): several clusters, stream-K off / on
for sk in -1 1; do
for cta in 0 72 146; do
  echo "== stream_k $sk CTA $cta"
  TRACE_CTA=$cta timeout 300 python tools/trace_tiles.py 3840x3840x3840 f32 "{\"config\": \"pair_256x256_k128\", \"stream_k\": $sk}" | grep -v "host enqueue\|columns"
done
done
