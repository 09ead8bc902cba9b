for c in 1 5; do python tools/trace_tiles.py 1024x1024x1024 f16 "{\"config\": $c}" | head -4; done
python tools/trace_tiles.py 2048x2048x2048 f32 | head -4
for c in 1 5; do ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.avg.per_second -s 2 -c 1 --clock-control none --csv python tools/one_launch.py "{\"M\":1024,\"mode\":\"f16\",\"config\":$c}" 2>/dev/null | grep -E "duration|cycles_elapsed" | awk -F'","' '{print $13, $15}'; done
M=1024 VARIANTS='[{"mode":"f16","config":1},{"mode":"f16","config":5},{"mode":"f32","config":1},{"mode":"f32","config":5}]' ROUNDS=5 REPS=50 python tools/ab.py
