for v in '{"mode":"f32"}' '{"mode":"f32","wait_hint_ns":20000}' '{"mode":"f32","wait_hint_ns":2000}' '{"mode":"f16"}' '{"mode":"f16","wait_hint_ns":20000}'; do bash tools/ncu_metrics.sh "$v"; done
VARIANTS='[{"mode":"f32"},{"mode":"f32","wait_hint_ns":20000},{"mode":"f16"},{"mode":"f16","wait_hint_ns":20000}]' ROUNDS=6 python tools/ab.py
M=16384 VARIANTS='[{"mode":"f32"},{"mode":"f32","wait_hint_ns":20000}]' ROUNDS=4 REPS=5 python tools/ab.py
