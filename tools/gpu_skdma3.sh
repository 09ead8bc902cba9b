#!/bin/bash
M=1024 VARIANTS='[{"mode":"f16","config":"splitk_128x256_s4"},{"mode":"f16","config":"splitk_128x256_s4","beta":0},{"mode":"f32","config":"splitk_128x256_s4","c_reduce":-1},{"mode":"f32","config":"splitk_128x256_s4","c_reduce":-1,"beta":0},{"mode":"f16","config":"solo_128x64"}]' ROUNDS=5 REPS=200 timeout 300 python tools/ab.py
