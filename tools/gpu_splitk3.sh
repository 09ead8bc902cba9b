#!/bin/bash
for d in 0 4 8 16 28; do python tools/trace_splitk.py 1024x1024x1024:f16:splitk_128x256_s4:$d 256x256x256:f16:splitk_128x256_s2:$d 1024x1024x1024:f32:splitk_128x256_s4:$d; done
