#!/bin/bash
SHAPES=1024x1024x4096,1024x1024x8192,512x512x8192,256x1024x16384,512x512x2048 CFGS=0,10,11,12 timeout 600 python tools/graph_bench.py
SHAPES=512x512x8192,256x1024x16384,512x512x2048,256x256x4096 CFGS=12 OPTS='{"c_reduce":-1}' timeout 600 python tools/graph_bench.py
