#!/bin/bash
VARIANTS='[{"mode":"f16"},{"mode":"f16","group_m":4},{"mode":"f16","group_m":16},{"mode":"f32"},{"mode":"f32","group_m":4},{"mode":"f32","group_m":16}]' ROUNDS=6 SECS=0.3 timeout 900 python tools/ab_power.py
VARIANTS='[{"mode":"f16"},{"mode":"f16","group_m":16},{"mode":"f16","group_m":32},{"mode":"f32"},{"mode":"f32","group_m":16}]' M=16384 ROUNDS=4 SECS=0.4 timeout 900 python tools/ab_power.py
