#!/bin/bash
for s in 8192x1024x1024 8192x1000x1000 8192x1000x1024 8192x1024x1000; do
  echo "== $s"
  timeout 300 python tools/trace_tiles.py $s f32 '{"config": "pair_256x256"}' | grep -v "host enqueue\|columns"
done
